mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "tiny_and_odd or batched" > gpurun_out/t.log 2>&1; echo rc=$? >> gpurun_out/t.log
