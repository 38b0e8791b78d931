# Round-2 profiling evidence, second pass (after the depth-first WSPD and the windowed
# CSR): one gpurun call; each ncu pass only after the same command exited 0 without
# ncu.  Summarised into profiles/ by tools/ncu_summary.py and tools/launch_summary.py.
set -u
mkdir -p gpurun_out
python tools/fe_once.py 100000 1.0 0.01 > gpurun_out/fe_cfg2.log 2>&1; echo fe_cfg2_rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv \
  -s 87 -c 87 python tools/fe_once.py 100000 1.0 0.01 > gpurun_out/ncu_list_cfg2.log 2>&1; echo list_cfg2_rc=$?
K='regex:k_refine|k_wspd_dfs|k_tree_coop|k_tree_local|k_sp_short_rows|k_sp_med_rows'
ncu --set full --clock-control none --import-source on -k "$K" -s 7 -c 7 -o gpurun_out/r02b_cfg2_top -f \
  python tools/fe_once.py 100000 1.0 0.01 > gpurun_out/ncu_cfg2_top.log 2>&1; echo full_cfg2_rc=$?
python tools/fe_once.py 100000 16.0 0.001 > gpurun_out/fe_cfg5w.log 2>&1; echo fe_cfg5w_rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5w.csv \
  -s 88 -c 88 python tools/fe_once.py 100000 16.0 0.001 > gpurun_out/ncu_list_cfg5w.log 2>&1; echo list_cfg5w_rc=$?
K5='regex:k_wspd_dfs|k_sp_'
ncu --set full --clock-control none --import-source on -k "$K5" -s 9 -c 9 -o gpurun_out/r02b_cfg5w_top -f \
  python tools/fe_once.py 100000 16.0 0.001 > gpurun_out/ncu_cfg5w_top.log 2>&1; echo full_cfg5w_rc=$?
