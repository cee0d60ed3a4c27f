mkdir -p gpurun_out/rst
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/rst/pytest.log 2>&1; echo rc=$? >> gpurun_out/rst/pytest.log
TSB_BENCH_FANOUT=inputs TSB_BENCH_SAME_DEVICE=1 TSB_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29530 bench.py --gpus 2 --steps 256 --warmup 8 > gpurun_out/rst/bench_inputs.json 2> gpurun_out/rst/bench_inputs.err
