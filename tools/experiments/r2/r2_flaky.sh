#!/bin/bash
out=gpurun_out/flaky; mkdir -p $out
for i in 1 2 3; do
  timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -o faulthandler_timeout=300 > $out/run_$i.log 2>&1
  echo "run $i rc=$? $(tail -1 $out/run_$i.log)"
done | tee $out/summary.txt
grep -h "^FAILED\|^ERROR" $out/run_*.log | sort | uniq -c
