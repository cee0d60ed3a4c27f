#!/bin/bash
# BASELINE configs on one GPU: per-batch launches and the persistent producer, ring above L2
out=gpurun_out/${1:-cfg}; mkdir -p $out
timeout 900 python tools/bench_configs.py --slots 80 > $out/configs.jsonl 2> $out/configs.err
timeout 600 python tools/bench_configs.py --only c1,c5video,c5llm --slots 80 --persistent > $out/configs_persistent.jsonl 2> $out/configs_persistent.err
