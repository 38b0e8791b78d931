mkdir -p gpurun_out
for cfg in "100000 16.0 0.001" "100000 4.0 0.001" "100000 1.0 0.01"; do python tools/fe_once.py $cfg 3; done > gpurun_out/fe6.log 2>&1
python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -q -x -k "cfg5 or sharded or shards or fused_csr or batch or csr" > gpurun_out/t6.log 2>&1; echo rc=$? >> gpurun_out/t6.log
