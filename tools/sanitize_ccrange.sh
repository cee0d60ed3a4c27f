#!/bin/bash
# compute-sanitizer over the persistent range kernel's parity tests (small geometries)
out=gpurun_out/${1:-san_ccrange}; mkdir -p $out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 1500 $CS --tool $tool --target-processes all --print-limit 20 --error-exitcode 9 \
      python -m pytest tests/test_gpu_crc_fused.py -q -p no:cacheprovider \
      -k "persistent and not full_c2" > $out/$tool.log 2>&1
  echo "$tool rc=$?" >> $out/summary.txt
done
