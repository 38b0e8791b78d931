mkdir -p gpurun_out
for st in 6 4 6 4; do timeout 600 python bench.py --steps 20 --warmup 5 --no-extras --streams $st > gpurun_out/bench_q.json 2> /dev/null; python -c "
import json
d=json.loads(open('gpurun_out/bench_q.json').read().strip().splitlines()[-1])
print('streams $st', 'value',round(d['value']),'e2e',round(d['e2e']['value']), d['e2e']['reps_ms'])
"; done > gpurun_out/bq.log 2>&1
