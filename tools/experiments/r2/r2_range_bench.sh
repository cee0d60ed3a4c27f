#!/bin/bash
bash tools/sanitize_ccrange.sh san_ccrange
out=gpurun_out/range_bench; mkdir -p $out
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo "rc=$?" >> $out/bench.err
timeout 900 python bench.py --persistent off --no-cpu-baseline > $out/bench_perbatch.json 2> $out/bench_perbatch.err
cat gpurun_out/san_ccrange/summary.txt; tail -c 600 $out/bench.json
