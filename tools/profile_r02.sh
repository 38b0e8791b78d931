# Round-2 profiling evidence (one gpurun call; each ncu pass only after the same
# command exited 0 without ncu).  Outputs land in gpurun_out/ and are summarised
# into profiles/ by tools/ncu_summary.py.
set -u
mkdir -p gpurun_out
python tools/fe_once.py 100000 1.0 0.01 > gpurun_out/fe_cfg2.log 2>&1; echo fe_cfg2_rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv \
  -s 90 python tools/fe_once.py 100000 1.0 0.01 > gpurun_out/ncu_list_cfg2.log 2>&1; echo list_cfg2_rc=$?
K='regex:k_refine|k_rwmd_f32|k_wspd_coop|k_tree_coop|k_tree_local|k_sp_|k_csr_'
ncu --set full --clock-control none --import-source on -k "$K" -s 12 -c 14 -o gpurun_out/r02_cfg2_top \
  python tools/fe_once.py 100000 1.0 0.01 > gpurun_out/ncu_cfg2_top.log 2>&1; echo full_cfg2_rc=$?
python tools/fe_once.py 100000 16.0 0.001 > gpurun_out/fe_cfg5w.log 2>&1; echo fe_cfg5w_rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5w.csv \
  -s 90 python tools/fe_once.py 100000 16.0 0.001 > gpurun_out/ncu_list_cfg5w.log 2>&1; echo list_cfg5w_rc=$?
K5='regex:k_wspd_coop|k_sp_|k_csr_'
ncu --set full --clock-control none --import-source on -k "$K5" -s 12 -c 12 -o gpurun_out/r02_cfg5w_top \
  python tools/fe_once.py 100000 16.0 0.001 > gpurun_out/ncu_cfg5w_top.log 2>&1; echo full_cfg5w_rc=$?
python tools/brute_once.py 1000000 > gpurun_out/brute_1m.log 2>&1; echo brute_rc=$?
ncu --set full --clock-control none --import-source on -k 'regex:k_rwmd_f32' -c 2 -o gpurun_out/r02_brute_1m \
  python tools/brute_once.py 1000000 > gpurun_out/ncu_brute.log 2>&1; echo full_brute_rc=$?
