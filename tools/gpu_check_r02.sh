mkdir -p gpurun_out
W1G_TIMING=1 python tools/fe_once.py 1000000 1.0 0.01 2 > gpurun_out/timing_1m.log 2>&1
ncu --set full --clock-control none --import-source on -k 'regex:k_sp_long_bitmap|k_sp_scatter|k_wspd_coop' -s 3 -c 3 -o gpurun_out/r02_cfg5w_csr \
  python tools/fe_once.py 100000 16.0 0.001 > gpurun_out/ncu_cfg5w_csr.log 2>&1; echo rc=$?
