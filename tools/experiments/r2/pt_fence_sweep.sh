set -x
for fd in "0 1" "1 1" "0 4" "1 4" "1 8"; do set -- $fd; for p in 4 8; do TSB_PT_FENCE=$1 TSB_PT_DEFER=$2 TSB_PT_PER_SM=$p timeout 200 python tools/pt_floor_probe.py 80 1024; done; done > gpurun_out/pt_fence.jsonl 2> gpurun_out/pt_fence.err
TSB_PT_FENCE=1 TSB_PT_DEFER=8 timeout 300 python -m pytest -q -x tests/test_gpu_pipeline.py -k "persistent" > gpurun_out/pt_tests.txt 2>&1
TSB_PT_FENCE=1 TSB_PT_DEFER=4 timeout 300 python -m pytest -q -x tests/test_gpu_pipeline.py -k "persistent" >> gpurun_out/pt_tests.txt 2>&1
tail -3 gpurun_out/pt_tests.txt
