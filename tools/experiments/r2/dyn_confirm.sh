timeout 600 python -m pytest -q -x tests/test_gpu_pipeline.py tests/test_gpu_crc_fused.py -p no:cacheprovider > gpurun_out/dyn2_tests.txt 2>&1
tail -1 gpurun_out/dyn2_tests.txt
for ep in 1 8 1 8; do TSB_EPOCHS_PER_LAUNCH=$ep PROBE_ONLY=c5llm,c1 timeout 200 python tools/pt_floor_probe.py 80 4096 | sed "s/}/, \"epl\": $ep}/"; done > gpurun_out/dyn_epl.jsonl 2> gpurun_out/dyn_epl.err
for p in 4 8; do TSB_PT_PER_SM=$p PROBE_ONLY=c5llm,c1 timeout 200 python tools/pt_floor_probe.py 80 4096 | sed "s/}/, \"per_sm_set\": $p}/"; done >> gpurun_out/dyn_epl.jsonl 2>> gpurun_out/dyn_epl.err
