#!/bin/bash
# fused-checksum A/B: the crc tests in both kernel modes, then per-batch timing for modes 0/1/2
out=gpurun_out/${1:-ccdbg}; mkdir -p $out; shift
for m in 1 2; do TSB_CRC_FUSED=$m timeout 600 python -m pytest tests/test_gpu_crc_fused.py -q -x -o faulthandler_timeout=240 > $out/pytest_mode$m.log 2>&1; echo "rc=$?" >> $out/pytest_mode$m.log; done
for m in ${@:-1 2 0}; do TSB_CRC_FUSED=$m timeout 300 python tools/crc_fused_timing.py f32,bf16,u8 200 | sed "s/^{/{\"mode\": $m, /" >> $out/timing.jsonl 2>> $out/timing.err; done
