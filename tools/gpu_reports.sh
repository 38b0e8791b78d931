# config reports (cfg1, cfg3, cfg4, cfg5) + the GPU tests, one gpurun call
timeout 900 python -m pytest tests -m gpu -x -q -k "row_shards or radix or row_classes" > gpurun_out/pytest_new.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_new.log
for c in cfg1 cfg3 cfg4 cfg5; do
  timeout 1200 python tools/report_configs.py $c --oracle > gpurun_out/report_$c.jsonl 2> gpurun_out/report_$c.err; echo $c rc=$?
  tail -c 600 gpurun_out/report_$c.err
done
