mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
for i in 1 2; do timeout 600 python bench.py --steps 20 --warmup 5 --no-extras > gpurun_out/bench_q.json 2> /dev/null; python -c "
import json
d=json.loads(open('gpurun_out/bench_q.json').read().strip().splitlines()[-1])
print('value',round(d['value']),'e2e',round(d['e2e']['value']), d['e2e']['reps_ms'])
"; done > gpurun_out/bq.log 2>&1
W1G_BATCH_TRACE=1 timeout 300 python tools/micro/e2e_trace.py > gpurun_out/e2e_trace.log 2>&1
