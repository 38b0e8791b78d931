mkdir -p gpurun_out
{
for o in 1 0; do echo "WSPD_OWNERS=$o"; for cfg in "100000 1.0 0.01 5" "100000 16.0 0.001 3" "100000 4.0 0.001 3" "1000000 1.0 0.01 3"; do W1G_WSPD_OWNERS=$o python tools/fe_once.py $cfg; done; done
} > gpurun_out/sweep2.log 2>&1
python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -q -x -k "cfg5 or fused_csr or stages or large or cfg3 or cfg4 or shard or deep" > gpurun_out/t12.log 2>&1; echo rc=$? >> gpurun_out/t12.log
W1G_BATCH_TRACE=1 python tools/e2e_probe.py 32 4 > gpurun_out/e2e_probe2.log 2>&1
