mkdir -p gpurun_out
{
for cfg in "100000 1.0 0.01 21" "20000 1.0 0.01 21" "100000 4.0 0.001 11" "100000 16.0 0.001 11"; do timeout 120 python tools/fe_once.py $cfg | head -1; done
} > gpurun_out/lt.log 2>&1
python tools/launch_rate.py 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except: continue
    if d['streams'] in (4,6,8): print(d['n'], d['streams'], round(d['pairs_per_s_device_makespan']))
" >> gpurun_out/lt.log 2>&1
