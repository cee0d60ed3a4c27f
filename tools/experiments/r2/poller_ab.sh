timeout 600 python -m pytest -q -x tests/test_gpu_pipeline.py > gpurun_out/poller_tests.txt 2>&1
tail -1 gpurun_out/poller_tests.txt
for pl in 1 0 1 0; do TSB_PT_POLLER=$pl timeout 200 python tools/pt_floor_probe.py 80 2048 | sed "s/}/, \"poller\": $pl}/"; done > gpurun_out/poller_ab.jsonl 2> gpurun_out/poller_ab.err
TSB_EPOCHS_PER_LAUNCH=8 timeout 200 python tools/pt_floor_probe.py 80 2048 | sed "s/}/, \"poller\": 1, \"epl\": 8}/" >> gpurun_out/poller_ab.jsonl 2>> gpurun_out/poller_ab.err
PROBE_ONLY=c1 TSB_PT_TRACE=3 timeout 200 python tools/pt_floor_probe.py 80 512 > gpurun_out/poller_trace_c1.txt 2>&1
