timeout 600 python -m pytest -q -x tests/test_gpu_pipeline.py tests/test_gpu_crc_fused.py > gpurun_out/pt_v2_tests.txt 2>&1
tail -2 gpurun_out/pt_v2_tests.txt
for p in 2 4 8; do TSB_PT_PER_SM=$p timeout 200 python tools/pt_floor_probe.py 80 1024; done > gpurun_out/pt_v2.jsonl 2> gpurun_out/pt_v2.err
PROBE_ONLY=c5llm TSB_PT_TRACE=4 TSB_PT_PER_SM=8 timeout 200 python tools/pt_floor_probe.py 80 256 > gpurun_out/pt_v2_trace_llm.txt 2>&1
