mkdir -p gpurun_out
for cm in 1 2 1 2; do W1G_BATCH_COMPACT=$cm timeout 600 python bench.py --steps 20 --warmup 5 --no-extras > gpurun_out/bench_q.json 2> /dev/null; python -c "
import json
d=json.loads(open('gpurun_out/bench_q.json').read().strip().splitlines()[-1])
print('compact $cm', 'value',round(d['value']),'e2e',round(d['e2e']['value']), d['e2e']['reps_ms'])
"; done > gpurun_out/bq.log 2>&1
W1G_BATCH_COMPACT=2 timeout 600 python -m pytest tests/test_gpu_parity.py -q -k batched > gpurun_out/c2test.log 2>&1; echo rc=$? >> gpurun_out/c2test.log
