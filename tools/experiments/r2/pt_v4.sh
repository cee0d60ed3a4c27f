timeout 900 python -m pytest -q -x tests/test_gpu_pipeline.py tests/test_gpu_crc_fused.py tests/test_gpu_control.py > gpurun_out/pt_v4_tests.txt 2>&1
tail -2 gpurun_out/pt_v4_tests.txt
for ep in 8 1; do for p in 4 8; do TSB_EPOCHS_PER_LAUNCH=$ep TSB_PT_PER_SM=$p timeout 200 python tools/pt_floor_probe.py 80 2048 | sed "s/}/, \"epl\": $ep}/"; done; done > gpurun_out/pt_v4.jsonl 2> gpurun_out/pt_v4.err
timeout 300 python bench.py --steps 512 --warmup 8 --no-cpu-baseline > gpurun_out/pt_v4_bench.json 2> gpurun_out/pt_v4_bench.err
