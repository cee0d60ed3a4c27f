#!/bin/bash
# ncu: persistent range fused kernel vs the per-batch fused kernel (u8 and f32)
out=gpurun_out/ncu_range; mkdir -p $out
for kind in ${KINDS:-u8 f32}; do
  TIMING_PERSIST=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:collate_crc_range -s 0 -c 1 \
      -o /tmp/rng_$kind -f python tools/crc_fused_timing.py $kind 16 > $out/rng_$kind.log 2>&1
  python tools/ncu_summary.py /tmp/rng_$kind.ncu-rep 20 > $out/ncu_range_$kind.txt 2>&1
  ncu -i /tmp/rng_$kind.ncu-rep --page raw --csv > $out/raw_range_$kind.csv 2>/dev/null
  ncu -i /tmp/rng_$kind.ncu-rep --page source --csv > $out/src_range_$kind.csv 2>/dev/null
  TIMING_PERSIST=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:collate_crc_kernel -s 10 -c 1 \
      -o /tmp/pb_$kind -f python tools/crc_fused_timing.py $kind 16 > $out/pb_$kind.log 2>&1
  python tools/ncu_summary.py /tmp/pb_$kind.ncu-rep 20 > $out/ncu_perbatch_$kind.txt 2>&1
  ncu -i /tmp/pb_$kind.ncu-rep --page raw --csv > $out/raw_perbatch_$kind.csv 2>/dev/null
done
