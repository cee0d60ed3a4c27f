#!/bin/bash
out=gpurun_out/bench_free; mkdir -p $out
for rep in 1 2; do for F in 0 12 8; do
  TSB_CC_RANGE_FREE_SMS=$F timeout 900 python bench.py --no-cpu-baseline > $out/b_${F}_$rep.json 2> /dev/null
  python -c "
import json; d=json.load(open('$out/b_${F}_$rep.json')); r=d['roofline']
print('free', $F, 'rep', $rep, d['value'], d['ms_per_step'], r['frac'], d['extra']['bf16']['avg_launch_ms'])"
done; done | tee $out/summary.txt
