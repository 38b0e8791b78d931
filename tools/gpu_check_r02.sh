mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/gpu_all2.log 2>&1; echo rc=$? >> gpurun_out/gpu_all2.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench4.json 2> gpurun_out/bench4.err; echo bench_rc=$?
