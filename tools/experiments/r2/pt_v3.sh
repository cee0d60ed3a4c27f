timeout 600 python -m pytest -q -x tests/test_gpu_pipeline.py tests/test_gpu_crc_fused.py > gpurun_out/pt_v3_tests.txt 2>&1
tail -2 gpurun_out/pt_v3_tests.txt
for p in 4 8; do TSB_PT_PER_SM=$p timeout 200 python tools/pt_floor_probe.py 80 1024; done > gpurun_out/pt_v3.jsonl 2> gpurun_out/pt_v3.err
TSB_EPOCHS_PER_LAUNCH=1 TSB_PT_PER_SM=8 PROBE_ONLY=c5llm timeout 200 python tools/pt_floor_probe.py 80 1024 >> gpurun_out/pt_v3.jsonl 2>> gpurun_out/pt_v3.err
TSB_PT_PER_SM=8 PROBE_ONLY=c5llm timeout 200 python tools/pt_floor_probe.py 80 4096 >> gpurun_out/pt_v3.jsonl 2>> gpurun_out/pt_v3.err
