#!/bin/bash
# one ncu --set full capture with the per-instruction source page kept (CSV)
# usage: bash tools/experiments/r2/r2_ncu_src.sh <outdir> <target> <kernel-regex> [env...]
out=gpurun_out/$1; mkdir -p $out; t=$2; k=$3; shift 3
env "$@" timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
    -o /tmp/src_$t -f python tools/profile_r2.py $t 6 > $out/$t.log 2>&1
python tools/ncu_summary.py /tmp/src_$t.ncu-rep 25 > $out/ncu_full_$t.txt 2>&1
ncu -i /tmp/src_$t.ncu-rep --page source --csv --print-source=sass > $out/src_$t.csv 2>/dev/null
ncu -i /tmp/src_$t.ncu-rep --page raw --csv > $out/raw_$t.csv 2>/dev/null
rm -f /tmp/src_$t.ncu-rep
