mkdir -p gpurun_out
W1G_TIMING=1 python tools/rwmd_breakdown.py 1000000 > gpurun_out/rwmd_1m.log 2>&1
W1G_TIMING=1 python tools/rwmd_breakdown.py 100000 > gpurun_out/rwmd_100k.log 2>&1
ncu --set full --clock-control none --import-source on -k 'regex:k_refine|k_rwmd_f32' -s 4 -c 4 -o gpurun_out/r02_cfg2_rwmd_b \
  python tools/fe_once.py 100000 1.0 0.01 > gpurun_out/ncu_cfg2_rwmd_b.log 2>&1; echo rwmd_rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2_b.csv \
  -s 95 python tools/fe_once.py 100000 1.0 0.01 > gpurun_out/ncu_list_cfg2_b.log 2>&1; echo list_rc=$?
python bench.py --steps 20 --warmup 5 > gpurun_out/bench6.json 2> gpurun_out/bench6.err; echo bench_rc=$?
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench6_ref.json 2> gpurun_out/bench6_ref.err; echo ref_rc=$?
