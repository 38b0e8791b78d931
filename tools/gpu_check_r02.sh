mkdir -p gpurun_out
{
for cfg in "100000 1.0 0.01 21" "20000 1.0 0.01 21" "100000 4.0 0.001 11" "100000 16.0 0.001 11"; do timeout 120 python tools/fe_once.py $cfg | grep -E "^n=|wspd" | sed "s/.*'wspd': \([0-9.]*\).*/wspd \1/" ; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_wspd_dfs --log-file gpurun_out/dfs2.csv python tools/fe_once.py 100000 1.0 0.01 > /dev/null 2>&1
grep k_wspd_dfs gpurun_out/dfs2.csv | awk -F'","' '{print "dfs cfg2", $NF}' | tail -1
} > gpurun_out/lt.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
