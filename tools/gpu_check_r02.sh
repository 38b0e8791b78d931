mkdir -p gpurun_out
for cfg in "100000 16.0 0.001 3" "100000 4.0 0.001 3" "100000 1.0 0.01 5" "1000000 1.0 0.01 3"; do python tools/fe_once.py $cfg; done > gpurun_out/fe19.log 2>&1
python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -q -x -k "cfg5 or fused or stages or large or cfg3 or deep or csr" > gpurun_out/t19.log 2>&1; echo rc=$? >> gpurun_out/t19.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5w_f.csv \
  -s 100 python tools/fe_once.py 100000 16.0 0.001 > gpurun_out/ncu_list_cfg5w_f.log 2>&1; echo list_rc=$?
