mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
for v in 1 0 1 0; do W1G_HOST_TAILS=$v timeout 300 python tools/micro/e2e_single_breakdown.py 2>&1 | head -1 | sed "s/^/host_tails=$v /"; done > gpurun_out/e2e1.log 2>&1
