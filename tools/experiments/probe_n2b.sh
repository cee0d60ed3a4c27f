mkdir -p gpurun_out/n2b
for f in inputs outputs; do
TSB_BENCH_FANOUT=$f TSB_BENCH_SAME_DEVICE=1 TSB_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29520 bench.py --gpus 2 --steps 256 --warmup 8 > gpurun_out/n2b/bench_$f.json 2> gpurun_out/n2b/bench_$f.err
done
timeout 600 python bench.py --no-cpu-baseline --steps 512 > gpurun_out/n2b/bench1.json 2> gpurun_out/n2b/bench1.err
