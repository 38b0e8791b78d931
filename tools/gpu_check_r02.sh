mkdir -p gpurun_out
for g in 1 0 1 0; do W1G_GRAPHS=$g timeout 600 python bench.py --steps 20 --warmup 5 --no-extras > gpurun_out/bench_q.json 2> /dev/null; python -c "
import json
d=json.loads(open('gpurun_out/bench_q.json').read().strip().splitlines()[-1])
print('graphs=$g value',round(d['value']),'e2e',round(d['e2e']['value']), d['e2e']['reps_ms'])
"; done > gpurun_out/bq.log 2>&1
