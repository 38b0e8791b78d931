# Round-2 profiling evidence, third pass (after the packed-source brute tile and the refine's
# FP32 warp median): the RWMD kernels' ncu captures that bench.py reads, and the cfg2 launch
# list.  Each ncu pass only after the same command exited 0 without ncu.  Summarised into
# profiles/ by tools/ncu_summary.py and tools/launch_summary.py.
set -u
mkdir -p gpurun_out
python tools/brute_once.py 1000000 > gpurun_out/brute_1m.log 2>&1; echo brute_rc=$?
ncu --set full --clock-control none --import-source on -k 'regex:k_rwmd_f32' -c 1 -o gpurun_out/r02c_brute_1m -f \
  python tools/brute_once.py 1000000 > gpurun_out/ncu_brute.log 2>&1; echo full_brute_rc=$?
python tools/fe_once.py 100000 1.0 0.01 > gpurun_out/fe_cfg2.log 2>&1; echo fe_cfg2_rc=$?
ncu --set full --clock-control none --import-source on -k 'regex:k_refine|k_rwmd_f32' -s 4 -c 4 \
  -o gpurun_out/r02c_cfg2_rwmd -f python tools/fe_once.py 100000 1.0 0.01 > gpurun_out/ncu_cfg2_rwmd.log 2>&1
echo full_rwmd_rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv \
  -s 87 -c 87 python tools/fe_once.py 100000 1.0 0.01 > gpurun_out/ncu_list_cfg2.log 2>&1; echo list_cfg2_rc=$?
