mkdir -p gpurun_out
python tools/report_configs.py cfg1 > gpurun_out/r02_cfg1_report.jsonl 2> gpurun_out/cfg1.err; echo cfg1_rc=$?
python tools/report_configs.py cfg4 > gpurun_out/r02_cfg4_report.jsonl 2> gpurun_out/cfg4.err; echo cfg4_rc=$?
python bench.py --workload cfg3 --steps 5 --warmup 3 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err; echo cfg3_rc=$?
python bench.py --workload cfg4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo b4_rc=$?
