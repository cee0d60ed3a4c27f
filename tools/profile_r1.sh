#!/bin/bash
out=gpurun_out/prof; mkdir -p $out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $out/launches_bench.csv \
    python bench.py --steps 32 --warmup 3 --no-cpu-baseline > $out/bench_under_ncu.log 2>&1
for k in f32 bf16 u8; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:collate_augment -s 2 -c 1 \
      -o $out/full_$k -f python tools/profile_one.py $k 4 > $out/full_$k.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:crc_kernel -s 1 -c 1 \
    -o $out/full_crc -f python tools/profile_one.py crc 3 > $out/full_crc.log 2>&1
