#!/bin/bash
# compute-sanitizer over the kernel parity tests (race detection)
out=gpurun_out/san; mkdir -p $out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 1200 $CS --tool $tool --target-processes all --print-limit 20 --error-exitcode 9 \
      python -m pytest tests/test_gpu_kernels.py tests/test_gpu_pipeline.py -q -x -p no:cacheprovider \
      -k "not cross_process" > $out/$tool.log 2>&1
  echo "$tool rc=$?" >> $out/summary.txt
done
