mkdir -p gpurun_out
{
for u in 1 2 4; do echo "U=$u"; for cfg in "100000 1.0 0.01 21" "100000 4.0 0.001 11" "100000 16.0 0.001 11"; do W1G_SP_SCATTER_U=$u timeout 120 python tools/fe_once.py $cfg; done; done
} > gpurun_out/bm.log 2>&1
for u in 1 4; do W1G_SP_SCATTER_U=$u ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_sp_scatter --log-file gpurun_out/scat_$u.csv python tools/fe_once.py 100000 16.0 0.001 > /dev/null 2>&1; done
timeout 900 python -m pytest tests -m gpu -x -q -k "cfg5 or parity" > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
