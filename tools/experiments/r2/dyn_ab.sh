TSB_PT_DYNAMIC=1 timeout 600 python -m pytest -q -x tests/test_gpu_pipeline.py -p no:cacheprovider > gpurun_out/dyn_tests.txt 2>&1
tail -1 gpurun_out/dyn_tests.txt
for d in 1 0 1 0; do TSB_PT_DYNAMIC=$d timeout 200 python tools/pt_floor_probe.py 80 2048 | sed "s/}/, \"dyn\": $d}/"; done > gpurun_out/dyn_ab.jsonl 2> gpurun_out/dyn_ab.err
TSB_PT_DYNAMIC=1 timeout 300 python tools/pt_launch_probe.py 6 > gpurun_out/dyn_launch.json 2>> gpurun_out/dyn_ab.err
