mkdir -p gpurun_out
timeout 1500 python tools/stress_r02.py 200 > gpurun_out/stress.log 2>&1; echo rc=$? >> gpurun_out/stress.log
for i in 1 2 3; do timeout 600 python bench.py --steps 10 --warmup 3 --no-extras > /dev/null 2>> gpurun_out/stress_bench.err; echo "bench $i rc=$?" >> gpurun_out/stress.log; done
