mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
{
for cfg in "100000 1.0 0.01 21" "20000 1.0 0.01 21" "1000000 1.0 0.01 5" "100000 16.0 0.001 11"; do timeout 120 python tools/fe_once.py $cfg | grep -E "^n=|split_tree" | sed 's/.*split_tree.: \([0-9.]*\).*/tree \1/' ; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_tree_local --log-file gpurun_out/tl.csv python tools/fe_once.py 100000 1.0 0.01 > /dev/null 2>&1
grep k_tree_local gpurun_out/tl.csv | awk -F'","' '{print "tree_local", $NF}' | tail -1
} > gpurun_out/lt.log 2>&1
