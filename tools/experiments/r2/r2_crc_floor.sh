#!/bin/bash
out=gpurun_out/${1:-crcfloor}; mkdir -p $out
for impl in tile v1; do
  TSB_CRC_IMPL=$impl timeout 300 python tools/crc_bench.py 154.14272 9.633792 2.1 0.4 > $out/crc_$impl.jsonl 2>&1
  TSB_CRC_IMPL=$impl TSB_CRC_INIT=none timeout 300 python tools/crc_bench.py 154.14272 9.633792 2.1 0.4 > $out/crc_${impl}_noinit.jsonl 2>&1
done
timeout 300 nsys --version > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:crc --csv --log-file $out/launches.csv python tools/crc_bench.py 2.1 > /dev/null 2>&1
