#!/bin/bash
# bf16 / u8 collate and the passthrough kernel at the final defaults: one full ncu capture each
out=gpurun_out/${PROF_OUT:-prof6}; mkdir -p $out
for k in bf16 u8; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:collate_augment -s 2 -c 1 \
      -o $out/full_$k -f python tools/profile_one.py $k 4 > $out/full_$k.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:passthrough -s 2 -c 1 \
    -o $out/full_passthrough -f python tools/profile_passthrough.py 5 > $out/full_pt.log 2>&1
