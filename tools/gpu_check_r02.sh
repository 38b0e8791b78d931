mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
for up in bulk per_pair bulk; do W1G_BATCH_UPLOAD=$up timeout 600 python bench.py --steps 20 --warmup 5 --no-extras > gpurun_out/bench_u.json 2> gpurun_out/bench_u.err; python -c "
import json
d=json.loads(open('gpurun_out/bench_u.json').read().strip().splitlines()[-1])
print('$up', 'value',round(d['value']),'e2e',round(d['e2e']['value']), d['e2e']['reps_ms'])
"; done > gpurun_out/bench_u.log 2>&1
timeout 300 python tools/micro/e2e_trace.py > gpurun_out/e2e_trace.log 2>&1
