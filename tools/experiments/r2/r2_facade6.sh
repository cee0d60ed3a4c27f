#!/bin/bash
out=gpurun_out/${1:-fr}; mkdir -p $out
for crc in 1 0; do TSB_FACADE_STATS=1 TSB_FR_CHECKSUM=$crc TSB_CONSUMERS=4 timeout 300 python tools/facade_rate.py 4000 >> $out/facade_rate.jsonl 2>> $out/facade_rate_$crc.err; done
