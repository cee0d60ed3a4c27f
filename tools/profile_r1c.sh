#!/bin/bash
# f32 collate at the current defaults: one full ncu capture
# + the launch list of the bench command
out=gpurun_out/${PROF_OUT:-prof3}; mkdir -p $out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:collate_augment -s 2 -c 1 \
    -o $out/full_f32 -f python tools/profile_one.py f32 4 > $out/full_f32.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $out/launches.csv python bench.py --steps 64 --warmup 4 --no-cpu-baseline > $out/b.log 2>&1
