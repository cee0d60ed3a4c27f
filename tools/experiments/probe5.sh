mkdir -p gpurun_out/p5
timeout 600 python -m pytest tests/test_gpu_group.py -x -q > gpurun_out/p5/pytest_group.log 2>&1; echo "rc=$?" >> gpurun_out/p5/pytest_group.log
timeout 600 python bench.py --no-cpu-baseline --steps 512 > gpurun_out/p5/bench1.json 2> gpurun_out/p5/bench1.err
TSB_BENCH_SAME_DEVICE=1 TSB_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 256 --warmup 8 > gpurun_out/p5/bench2.json 2> gpurun_out/p5/bench2.err
echo done
