# ncu --set full on the front end's top kernels (one launch each, warm front end), summary -> gpurun_out/ncu_top.jsonl
K='regex:k_wspd_coop|k_tree_coop|k_tree_local|k_refine|k_rwmd_f32|k_rs_onesweep|k_csr_med_rows|k_csr_short_rows|k_csr_scatter|k_csr_count|k_csr_emit|k_dc_snap|k_zc_emit'
W1G_OVERLAP=0 python tools/one_fe.py 100000 > gpurun_out/plain_top.log 2>&1 && \
W1G_OVERLAP=0 ncu --set full --clock-control none -k "$K" -s 26 -c 30 -o gpurun_out/prof_top python tools/one_fe.py 100000 > gpurun_out/ncu_top.log 2>&1
echo rc=$?
