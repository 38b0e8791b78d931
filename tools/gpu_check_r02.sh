mkdir -p gpurun_out
python -m pytest tests/test_gpu_configs.py -q -x -k "shard or gathered" > gpurun_out/t20.log 2>&1; echo rc=$? >> gpurun_out/t20.log
python bench.py --workload cfg3 --steps 5 --warmup 3 > gpurun_out/bench_cfg3b.json 2> gpurun_out/bench_cfg3b.err; echo cfg3_rc=$?
