# ncu evidence for the front end (one gpurun call; see B200_PROFILING.md)
B="python bench.py --profile-only --steps 1 --warmup 1 --no-w1 --no-cpu-baseline"
$B > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_list.log 2>&1
echo list_rc=$?
$B > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_rs_onesweep|k_refine}" -s ${KSKIP:-20} -c ${KCOUNT:-4} -o gpurun_out/prof_${KTAG:-misc} $B > gpurun_out/ncu_full.log 2>&1
echo full_rc=$?
tail -2 gpurun_out/ncu_full.log
