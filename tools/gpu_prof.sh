# ncu evidence for the front end (one gpurun call; see B200_PROFILING.md)
set -x
B="python bench.py --profile-only --steps 1 --warmup 1 --no-w1 --no-cpu-baseline"
./tools/rwmd_micro 100000 > gpurun_out/micro.json 2>&1; cat gpurun_out/micro.json
$B > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_list.log 2>&1
echo list_rc=$?
$B > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_rwmd_f32 -s 2 -c 1 -o gpurun_out/prof_rwmd $B > gpurun_out/ncu_full.log 2>&1
echo full_rc=$?
tail -3 gpurun_out/ncu_full.log
