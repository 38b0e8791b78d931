mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo rc=$?
bash tools/profile_r02b.sh > gpurun_out/profile_r02b.log 2>&1
