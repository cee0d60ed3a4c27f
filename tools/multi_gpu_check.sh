#!/bin/bash
# usage (on a multi-GPU box): bash tools/multi_gpu_check.sh <tag> [max_gpus]
# The §5 measurements this one-GPU round could not take: bench.py at N = 2, 4, 8
# with the two-stage (inputs) and fused output (outputs) all-gathers, and the
# NCCL comparison points, each rank on its own GPU over NVLink/NVSwitch.
tag=$1; max=${2:-8}; out=gpurun_out/$tag; mkdir -p $out
n=$(nvidia-smi -L | wc -l); [ "$n" -lt "$max" ] && max=$n
port=29600
for N in 2 4 8; do
  [ "$N" -gt "$max" ] && break
  for f in inputs outputs; do
    port=$((port + 1))
    TSB_BENCH_FANOUT=$f timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
      --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N \
      > $out/bench_n${N}_$f.json 2> $out/bench_n${N}_$f.err
  done
  port=$((port + 1))
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port $port tools/nccl_broadcast_compare.py \
    > $out/nccl_n$N.json 2> $out/nccl_n$N.err
done
NCCL_DEBUG=INFO timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $max \
  --master-addr 127.0.0.1 --master-port $((port + 1)) tools/nccl_broadcast_compare.py \
  2>&1 | grep -i "nvls\|NVLS" | head -20 > $out/nvls.txt
