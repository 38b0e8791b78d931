mkdir -p gpurun_out
bash tools/profile_r02.sh
python bench.py --steps 20 --warmup 5 > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo bench_rc=$?
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench3_ref.json 2> gpurun_out/bench3_ref.err; echo ref_rc=$?
