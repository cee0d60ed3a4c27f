timeout 600 python -m pytest -q -x tests/test_gpu_pipeline.py > gpurun_out/pt_v7_tests.txt 2>&1
tail -1 gpurun_out/pt_v7_tests.txt
for ep in 1 8 1 8; do TSB_EPOCHS_PER_LAUNCH=$ep timeout 200 python tools/pt_floor_probe.py 80 2048 | sed "s/}/, \"epl\": $ep}/"; done > gpurun_out/pt_v7.jsonl 2> gpurun_out/pt_v7.err
