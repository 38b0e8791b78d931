mkdir -p gpurun_out
{
for d in 1 0; do echo "DFS=$d"; for cfg in "100000 1.0 0.01 21" "100000 4.0 0.001 11" "100000 16.0 0.001 11"; do W1G_WSPD_DFS=$d timeout 120 python tools/fe_once.py $cfg; done; done
} > gpurun_out/dfs.log 2>&1
