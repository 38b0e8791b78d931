# front-end time with RWMD sequential (0), overlapped with emit+assemble (1) or with the whole back end (2)
for o in 0 1 2 3 4; do
  W1G_OVERLAP=$o python bench.py --steps 20 --warmup 5 --no-w1 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('overlap=$o', round(d['ms_per_step'],3), 'ms', {k: round(v,3) for k,v in d['stage_ms'].items()}, 'e2e', round(d['e2e']['ms_per_pair'],3))"
done
