#!/bin/bash
out=gpurun_out/${1:-launches_r2}; mkdir -p $out
TSB_BENCH_E2E_BATCHES=64 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file $out/launches_bench.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $out/bench_under_ncu.log 2>&1
