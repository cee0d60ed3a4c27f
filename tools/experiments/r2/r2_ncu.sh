#!/bin/bash
# round 2: one ncu --set full capture per kernel of the data plane (summarised
# on the box: gpurun copies back <= 64 MiB), plus the bench launch list
out=gpurun_out/${1:-ncu_r2}; mkdir -p $out
shift
targets=${@:-"f32crc bf16crc u8crc f32 bf16 u8 passthrough llm llm_persistent video rebatch fanout twostage_gather twostage_collate crc"}
declare -A K=( [f32crc]=collate_crc [bf16crc]=collate_crc [u8crc]=collate_crc [f32]=collate_augment [bf16]=collate_augment [u8]=collate_augment [passthrough]=passthrough_multi
  [llm]=passthrough_multi [llm_persistent]=persistent_passthrough [video]=passthrough_multi [rebatch]=rebatch_window
  [fanout]=fanout_v16 [twostage_gather]=passthrough_multi [twostage_collate]=collate_augment [crc]=crc_ )
declare -A W=( [twostage_gather]=twostage [twostage_collate]=twostage )
declare -A N=( [llm_persistent]="64 0" [rebatch]="4 1" [fanout]="4 1" [crc]="4 1" )
for t in $targets; do
  what=${W[$t]:-$t}; ns=${N[$t]:-"6 2"}; n=${ns% *}; skip=${ns#* }
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:${K[$t]} -s $skip -c 1 \
      -o /tmp/full_$t -f python tools/profile_r2.py $what $n > $out/$t.log 2>&1
  python tools/ncu_summary.py /tmp/full_$t.ncu-rep 20 > $out/ncu_full_$t.txt 2>&1
  ncu -i /tmp/full_$t.ncu-rep --page raw --csv > $out/raw_$t.csv 2>/dev/null
  rm -f /tmp/full_$t.ncu-rep
done
