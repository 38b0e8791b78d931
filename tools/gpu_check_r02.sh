mkdir -p gpurun_out
python -m pytest tests/test_gpu_retrieval.py tests/test_distributed.py -q -x > gpurun_out/t17.log 2>&1; echo rc=$? >> gpurun_out/t17.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench5.json 2> gpurun_out/bench5.err; echo bench_rc=$?
