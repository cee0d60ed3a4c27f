CONFIGS=1 bash tools/round_check.sh r2m
for i in $(seq 1 5); do timeout 300 python -m pytest -q -x tests/test_gpu_pipeline.py tests/test_gpu_crc_fused.py -k "persistent or range" -p no:cacheprovider 2>&1 | tail -1; done > gpurun_out/r2m/persistent_stress.txt
