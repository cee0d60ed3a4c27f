#!/bin/bash
# persistent range kernel: per-batch time with SMs left free for other kernels
out=gpurun_out; mkdir -p $out
for rep in 1 2; do
for F in ${FREE:-0 8 12 16 20 24}; do
  TSB_CC_RANGE_FREE_SMS=$F TIMING_PERSIST=1 timeout 120 python tools/crc_fused_timing.py ${KINDS:-f32,bf16,u8} 512 2>&1 | grep '"checksum": true' | sed "s/^{/{\"free_sms\": $F, \"rep\": $rep, /"
done; done | tee $out/range_free_sms2.jsonl
