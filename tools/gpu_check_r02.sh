mkdir -p gpurun_out
{
for cfg in "100000 16.0 0.001 15" "100000 1.0 0.01 21" "100000 4.0 0.001 15" "100000 8.0 0.001 15" "1000000 1.0 0.01 5"; do timeout 200 python tools/fe_once.py $cfg | grep -v "^{"; done
} > gpurun_out/bm.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
