CONFIGS=1 bash tools/round_check.sh r2j
for i in $(seq 1 10); do timeout 300 python -m pytest -q -x tests/test_gpu_pipeline.py -k "persistent" -p no:cacheprovider 2>&1 | tail -1; done > gpurun_out/r2j/persistent_stress.txt
