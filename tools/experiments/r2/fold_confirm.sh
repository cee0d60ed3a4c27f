timeout 600 python -m pytest -q -x tests/test_gpu_crc_fused.py tests/test_gpu_fullsize.py tests/test_gpu_fullsize_configs.py -p no:cacheprovider > gpurun_out/fold_confirm_tests.txt 2>&1
tail -1 gpurun_out/fold_confirm_tests.txt
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/fold_bench.json 2> gpurun_out/fold_bench.err
TIMING_PERSIST=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:collate_crc_range -s 1 -c 1 -o gpurun_out/rng_f32_fold -f python tools/crc_fused_timing.py f32 64 > gpurun_out/rng_f32_fold.log 2>&1
python tools/ncu_summary.py gpurun_out/rng_f32_fold.ncu-rep 20 > gpurun_out/ncu_full_range_f32_fold.txt 2>&1
rm -f gpurun_out/rng_f32_fold.ncu-rep
