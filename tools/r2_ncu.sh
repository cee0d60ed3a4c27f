#!/bin/bash
# round 2: one ncu --set full capture per kernel of the data plane, plus the bench launch list
out=gpurun_out/${1:-ncu_r2}; mkdir -p $out
cap() {  # name regex what n skip
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$2 -s $5 -c 1 \
      -o $out/full_$1 -f python tools/profile_r2.py $3 $4 > $out/$1.log 2>&1
}
cap f32 collate_augment f32 6 2
cap bf16 collate_augment bf16 6 2
cap u8 collate_augment u8 6 2
cap passthrough passthrough_multi passthrough 6 2
cap llm passthrough_multi llm 6 2
cap llm_persistent persistent_passthrough llm_persistent 64 0
cap video passthrough_multi video 6 2
cap rebatch rebatch_window rebatch 4 1
cap fanout fanout_v16 fanout 4 1
cap twostage_gather passthrough_multi twostage 6 2
cap twostage_collate collate_augment twostage 6 2
cap crc crc_tile crc 4 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file $out/launches_bench.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $out/bench_under_ncu.log 2>&1
