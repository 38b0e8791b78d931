mkdir -p gpurun_out
{
for d in 1 0; do echo "DFS=$d"; for cfg in "100000 1.0 0.01 5" "100000 4.0 0.001 3" "100000 16.0 0.001 3"; do W1G_WSPD_DFS=$d timeout 120 python tools/fe_once.py $cfg; done; done
} > gpurun_out/dfs.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
ncu --set full --clock-control none --import-source on -k 'regex:k_wspd_dfs' -s 1 -c 1 -o gpurun_out/dfs_cfg2 -f \
  python tools/fe_once.py 100000 1.0 0.01 > gpurun_out/ncu_dfs_cfg2.log 2>&1; echo rc=$?
ncu --set full --clock-control none --import-source on -k 'regex:k_wspd_dfs' -s 1 -c 1 -o gpurun_out/dfs_cfg5w -f \
  python tools/fe_once.py 100000 16.0 0.001 > gpurun_out/ncu_dfs_cfg5w.log 2>&1; echo rc=$?
