#!/bin/bash
out=gpurun_out/twostage_crc; mkdir -p $out
true
TSB_BENCH_BACKEND=gloo TSB_BENCH_SAME_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 64 --warmup 4 --no-cpu-baseline > $out/bench_n2.json 2> $out/bench_n2.err
echo "rc=$?" >> $out/bench_n2.err
cat $out/tests.txt; tail -c 1500 $out/bench_n2.json; tail -3 $out/bench_n2.err
