mkdir -p gpurun_out
for st in 4 6 4 6; do python bench.py --steps 20 --warmup 5 --streams $st --no-extras > gpurun_out/bench_q$st.json 2> gpurun_out/bench_q$st.err; python -c "
import json
d=json.loads(open('gpurun_out/bench_q$st.json').read().strip().splitlines()[-1])
print($st, 'value',round(d['value']),'e2e',round(d['e2e']['value']), d['e2e']['reps_ms'])
"; done > gpurun_out/bench_q.log 2>&1
