#!/bin/bash
# fused-checksum A/B: the crc tests, then per-batch timing with the fused kernel (1) and the output CRC (0)
out=gpurun_out/${1:-ccdbg}; mkdir -p $out; shift
timeout 600 python -m pytest tests/test_gpu_crc_fused.py -q -x -o faulthandler_timeout=240 > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
for m in ${@:-1}; do TSB_CRC_FUSED=$m timeout 300 python tools/crc_fused_timing.py f32,bf16,u8 200 | sed "s/^{/{\"mode\": $m, /" >> $out/timing.jsonl 2>> $out/timing.err; done
