#!/bin/bash
# persistent fused range: tests (bounded), then timing vs the per-batch fused kernel
out=gpurun_out/${1:-persist}; mkdir -p $out
timeout 300 python -m pytest tests/test_gpu_crc_fused.py -q -x -k "persistent" -o faulthandler_timeout=120 > $out/pytest_persist.log 2>&1; echo "rc=$?" >> $out/pytest_persist.log
if grep -q "rc=0" $out/pytest_persist.log; then
  for b in 256 512; do TIMING_B=$b TIMING_PERSISTENT=1 timeout 300 python tools/crc_fused_timing.py f32,bf16,u8 400 >> $out/timing.jsonl 2>> $out/timing.err; done
  timeout 600 python -m pytest tests/test_gpu_crc_fused.py -q -o faulthandler_timeout=200 > $out/pytest_all.log 2>&1; echo "rc=$?" >> $out/pytest_all.log
fi
