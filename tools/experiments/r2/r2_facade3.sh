#!/bin/bash
# facade through the public API (HBM store): checksum on (fused) / off, 1..16 consumers
out=gpurun_out/${1:-fr3}; mkdir -p $out
for crc in 1 0; do for k in 1 4 8 16; do
  TSB_FR_CHECKSUM=$crc TSB_CONSUMERS=$k timeout 300 python tools/facade_rate.py 3000 >> $out/facade_rate.jsonl 2>> $out/facade_rate.err
done; done
