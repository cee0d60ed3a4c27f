#!/bin/bash
out=gpurun_out/${1:-q}; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_control.py tests/test_gpu_crc_fused.py tests/test_gpu_facade.py -q -o faulthandler_timeout=300 > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
timeout 300 python tools/crc_fused_timing.py f32,bf16,u8 400 > $out/timing.jsonl 2> $out/timing.err
