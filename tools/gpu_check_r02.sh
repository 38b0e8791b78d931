mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_random_sweep.py -x -q > gpurun_out/sweep_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/sweep_tests.log
