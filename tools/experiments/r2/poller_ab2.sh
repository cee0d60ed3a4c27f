timeout 600 python -m pytest -q -x tests/test_gpu_pipeline.py > gpurun_out/poller2_tests.txt 2>&1
tail -1 gpurun_out/poller2_tests.txt
for pl in 1 0 1 0; do TSB_PT_POLLER=$pl timeout 200 python tools/pt_floor_probe.py 80 2048 | sed "s/}/, \"poller\": $pl}/"; done > gpurun_out/poller_ab2.jsonl 2> gpurun_out/poller_ab2.err
