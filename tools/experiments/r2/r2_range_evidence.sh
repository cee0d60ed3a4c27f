#!/bin/bash
# persistent range kernel evidence: the order-lifetime regression test without
# the fix (must fail), ncu --set full of a 56-batch range launch (f32/bf16/u8),
# and the bench launch list
out=gpurun_out/range_ev; mkdir -p $out
timeout 300 python - > $out/negative_check.txt 2>&1 <<'PY'
import pytest, paper_2409_18749_b200.ring as r
r.hold_for_stream = lambda a, s: None   # the fix disabled
rc = pytest.main(["-q", "-p", "no:cacheprovider", "tests/test_gpu_crc_fused.py", "-k", "outlive"])
print("pytest rc without hold_for_stream:", int(rc))
PY
for kind in f32 bf16 u8; do
  TIMING_PERSIST=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:collate_crc_range -s 1 -c 1 \
      -o /tmp/rng_$kind -f python tools/crc_fused_timing.py $kind 64 > $out/rng_$kind.log 2>&1
  python tools/ncu_summary.py /tmp/rng_$kind.ncu-rep 20 > $out/ncu_full_range_$kind.txt 2>&1
  ncu -i /tmp/rng_$kind.ncu-rep --page raw --csv > $out/raw_range_$kind.csv 2>/dev/null
done
TSB_BENCH_E2E_BATCHES=64 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file $out/launches_bench.csv python bench.py --steps 128 --warmup 5 --no-cpu-baseline > $out/bench_under_ncu.log 2>&1
echo "launches rc=$?" >> $out/bench_under_ncu.log
tail -3 $out/negative_check.txt; head -4 $out/ncu_full_range_f32.txt
