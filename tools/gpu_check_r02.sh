mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
{
for cfg in "100000 1.0 0.01 21" "1000000 1.0 0.01 7"; do timeout 200 python tools/fe_once.py $cfg | head -1; done
} > gpurun_out/bm.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_refine --log-file gpurun_out/refine.csv python tools/fe_once.py 100000 1.0 0.01 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_refine --log-file gpurun_out/refine1m.csv python tools/fe_once.py 1000000 1.0 0.01 > /dev/null 2>&1
