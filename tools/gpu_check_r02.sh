mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
W1G_DEBUG_NO_D2H=1 W1G_BATCH_COMPACT=0 timeout 300 python tools/micro/e2e_trace.py > gpurun_out/e2e_trace_nod2h.log 2>&1
W1G_GRAPHS=0 timeout 300 python tools/micro/e2e_trace.py > gpurun_out/e2e_trace.log 2>&1
