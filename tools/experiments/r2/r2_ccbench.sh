#!/bin/bash
# fused-checksum timing (tool, no consumers) + the default bench line
out=gpurun_out/${1:-ccb}; mkdir -p $out
timeout 300 python tools/crc_fused_timing.py f32,bf16,u8 400 > $out/timing.jsonl 2> $out/timing.err
timeout 600 python bench.py --no-cpu-baseline > $out/bench.json 2> $out/bench.err
