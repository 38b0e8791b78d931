mkdir -p gpurun_out
timeout 1200 python tools/stress_r02.py 60 > gpurun_out/stress.log 2>&1; echo rc=$? >> gpurun_out/stress.log
