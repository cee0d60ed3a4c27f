TIMING_PERSIST=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:collate_crc_range -s 1 -c 1 \
    -o gpurun_out/rng_f32 -f python tools/crc_fused_timing.py f32 64 > gpurun_out/rng_f32.log 2>&1
ncu -i gpurun_out/rng_f32.ncu-rep --page source --csv --print-source sass > gpurun_out/rng_f32_sass.csv 2>/dev/null
ls -la gpurun_out/rng_f32*
