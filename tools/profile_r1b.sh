#!/bin/bash
out=gpurun_out/prof2; mkdir -p $out
for k in f32 bf16 fanout2_bf16; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:collate_augment -s 2 -c 1 \
      -o $out/full_$k -f python tools/profile_one.py $k 4 > $out/full_$k.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:passthrough -s 2 -c 1 \
    -o $out/full_passthrough -f python tools/profile_passthrough.py 5 > $out/full_pt.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:crc_kernel -s 1 -c 1 \
    -o $out/full_crc -f python tools/profile_one.py crc 3 > $out/full_crc.log 2>&1
