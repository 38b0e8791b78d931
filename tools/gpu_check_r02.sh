mkdir -p gpurun_out
for cfg in "100000 16.0 0.001" "100000 4.0 0.001" "100000 1.0 0.01" "1000000 1.0 0.01"; do python tools/fe_once.py $cfg 3; done > gpurun_out/fe10.log 2>&1
python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -q -x -k "cfg5 or fused_csr or csr or stages or non_finite or cfg3 or cfg4 or deep" > gpurun_out/t10.log 2>&1; echo rc=$? >> gpurun_out/t10.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5w_e.csv \
  -s 90 python tools/fe_once.py 100000 16.0 0.001 > gpurun_out/ncu_list_cfg5w_e.log 2>&1; echo list_rc=$?
ncu --set full --clock-control none --import-source on -k 'regex:k_refine|k_rwmd_f32' -s 4 -c 4 -o gpurun_out/r02_cfg2_rwmd \
  python tools/fe_once.py 100000 1.0 0.01 > gpurun_out/ncu_cfg2_rwmd.log 2>&1; echo rwmd_rc=$?
