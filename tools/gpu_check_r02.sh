mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
{
for cfg in "100000 1.0 0.01 21" "100000 4.0 0.001 11" "100000 16.0 0.001 11" "1000000 1.0 0.01 5" "20000 1.0 0.01 21"; do timeout 120 python tools/fe_once.py $cfg; done
} > gpurun_out/bm.log 2>&1
python tools/launch_rate.py > gpurun_out/launch_rate_new.jsonl 2>&1
