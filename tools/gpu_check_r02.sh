mkdir -p gpurun_out
W1G_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 4 --warmup 3 > gpurun_out/bench_2r.json 2> gpurun_out/bench_2r.err; echo rc=$? >> gpurun_out/bench_2r.err
W1G_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > gpurun_out/bench_2r_ref.json 2> gpurun_out/bench_2r_ref.err; echo rc=$? >> gpurun_out/bench_2r_ref.err
