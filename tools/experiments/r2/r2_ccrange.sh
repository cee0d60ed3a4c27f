#!/bin/bash
# persistent fused collate+CRC range kernel: parity tests then timing A/B
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_crc_fused.py -x -q -k persistent 2>&1 | tail -15 > gpurun_out/ccrange_tests.txt
cat gpurun_out/ccrange_tests.txt
for P in 0 1; do
  TIMING_PERSIST=$P timeout 300 python tools/crc_fused_timing.py f32,bf16,u8 256 2>&1 | grep '^{' 
done | tee gpurun_out/ccrange_timing.jsonl
