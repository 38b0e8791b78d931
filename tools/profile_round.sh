# profiling evidence for profiles/ (one gpurun call): the bench line, a launch list of
# one warm cfg2 front end, and ncu --set full of its top kernels (each only after the
# same command exited 0 without ncu)
timeout 600 python bench.py > gpurun_out/bench_full.log 2>&1; echo bench_rc=$?
W1G_OVERLAP=0 python tools/one_fe.py 100000 > gpurun_out/plain_fe.log 2>&1 && \
W1G_OVERLAP=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_fe.csv \
  python tools/one_fe.py 100000 > gpurun_out/ncu_fe.log 2>&1; echo list_rc=$?
K='regex:k_wspd_coop|k_tree_coop|k_tree_local|k_refine|k_rwmd_f32|k_rs_onesweep|k_sp_|k_dc_snap|k_zc_emit'
W1G_OVERLAP=0 ncu --set full --clock-control none --import-source on -k "$K" -s 24 -c 30 -o gpurun_out/prof_top \
  python tools/one_fe.py 100000 > gpurun_out/ncu_top.log 2>&1; echo full_rc=$?
