mkdir -p gpurun_out/n2
timeout 600 python bench.py --no-cpu-baseline --steps 256 > gpurun_out/n2/bench1.json 2> gpurun_out/n2/bench1.err
TSB_BENCH_SAME_DEVICE=1 TSB_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 128 --warmup 8 > gpurun_out/n2/bench2.json 2> gpurun_out/n2/bench2.err
