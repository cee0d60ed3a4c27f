#!/bin/bash
out=gpurun_out/ccrange_dbg4; mkdir -p $out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 600 python -m pytest tests/test_gpu_crc_fused.py -q -p no:cacheprovider 2>&1 | tail -3 > $out/tests.txt
timeout 900 $CS --tool racecheck --print-limit 5 python tools/ccrange_diag.py > $out/race.txt 2>&1
bash tools/sanitize_ccrange.sh san_ccrange2
cat $out/tests.txt; tail -n 9 $out/race.txt; cat gpurun_out/san_ccrange2/summary.txt
