#!/bin/bash
out=gpurun_out/${1:-fr4}; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_control.py tests/test_gpu_facade.py tests/test_gpu_facade_multi.py tests/test_gpu_crc_fused.py -q -x -o faulthandler_timeout=300 > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
for k in 4 8; do TSB_FR_CHECKSUM=1 TSB_CONSUMERS=$k timeout 300 python tools/facade_rate.py 3000 >> $out/facade_rate.jsonl 2>> $out/facade_rate.err; done
timeout 600 python bench.py --no-cpu-baseline --steps 64 > $out/bench.json 2> $out/bench.err
