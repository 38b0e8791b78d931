mkdir -p gpurun_out
for cfg in "100000 16.0 0.001" "100000 4.0 0.001" "100000 1.0 0.01" "1000000 1.0 0.01"; do python tools/fe_once.py $cfg 3; done > gpurun_out/fe8.log 2>&1
python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -q -x -k "cfg5 or fused_csr or csr or stages or non_finite or cfg3 or cfg4" > gpurun_out/t8.log 2>&1; echo rc=$? >> gpurun_out/t8.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5w_c.csv \
  -s 90 python tools/fe_once.py 100000 16.0 0.001 > gpurun_out/ncu_list_cfg5w_c.log 2>&1; echo list_rc=$?
for st in 4 6 8; do python bench.py --steps 8 --warmup 3 --no-extras --streams $st > gpurun_out/bench_s$st.json 2>&1; done
