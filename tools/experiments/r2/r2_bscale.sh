#!/bin/bash
# per-batch time vs batch size (fused checksum kernel and the plain collate): a + b*B
out=gpurun_out/${1:-bscale}; mkdir -p $out
for b in 128 256 512; do TIMING_B=$b timeout 300 python tools/crc_fused_timing.py f32,bf16 200 >> $out/timing.jsonl 2>> $out/timing.err; done
