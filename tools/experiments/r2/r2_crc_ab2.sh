#!/bin/bash
out=gpurun_out/${1:-crcab2}; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -k crc > $out/pytest_rows.log 2>&1; echo "rc=$?" >> $out/pytest_rows.log
TSB_CRC_IMPL=tile timeout 600 python -m pytest tests/test_gpu_kernels.py -q -k crc > $out/pytest_tile.log 2>&1; echo "rc=$?" >> $out/pytest_tile.log
for impl in rows tile v1; do
  TSB_CRC_IMPL=$impl timeout 300 python tools/crc_bench.py 154.14272 77.07 38.5 9.633792 2.1 > $out/crc_$impl.jsonl 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:crc_rows -s 1 -c 1 \
    -o $out/full_crc_rows -f python tools/profile_r2.py crc 4 > $out/ncu_crc.log 2>&1
