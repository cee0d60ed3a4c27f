#!/bin/bash
# facade with the checksum at several buffer depths; producer step profile
out=gpurun_out/${1:-fr}; mkdir -p $out
for d in 6 12; do TSB_FR_DEPTH=$d TSB_FR_CHECKSUM=1 TSB_CONSUMERS=4 timeout 300 python tools/facade_rate.py 4000 >> $out/facade_rate.jsonl 2>> $out/facade_rate.err; done
TSB_FR_CHECKSUM=0 TSB_CONSUMERS=4 timeout 300 python tools/facade_rate.py 4000 >> $out/facade_rate.jsonl 2>> $out/facade_rate.err
