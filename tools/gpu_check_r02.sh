mkdir -p gpurun_out
timeout 300 python tools/micro/sync_latency.py > gpurun_out/sync_latency.log 2>&1; echo rc=$?
