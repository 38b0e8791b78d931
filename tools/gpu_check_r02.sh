mkdir -p gpurun_out
W1G_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 4 --warmup 3 --no-extras > gpurun_out/bench_2r.json 2> gpurun_out/bench_2r.err; echo rc=$? >> gpurun_out/bench_2r.err
timeout 600 python bench.py --steps 5 --warmup 3 --no-extras > gpurun_out/bench_1r.json 2> gpurun_out/bench_1r.err; echo rc=$? >> gpurun_out/bench_1r.err
