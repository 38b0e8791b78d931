mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_new.json 2> gpurun_out/bench_new.err; echo rc=$?
python tools/launch_rate.py > gpurun_out/launch_rate_new.jsonl 2>&1
