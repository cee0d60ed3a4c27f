#!/bin/bash
out=gpurun_out/${1:-ccdbg}; mkdir -p $out; shift
for d in ${@:-0 1 2 3}; do TSB_CC_DEBUG=$d timeout 300 python tools/crc_fused_timing.py f32,bf16 200 | grep '"checksum": true' | sed "s/^{/{\"dbg\": $d, /" >> $out/timing.jsonl 2>> $out/timing.err; done
