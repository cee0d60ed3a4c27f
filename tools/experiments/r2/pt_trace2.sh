PROBE_ONLY=c5llm TSB_PT_TRACE=4 TSB_PT_PER_SM=4 timeout 200 python tools/pt_floor_probe.py 80 256 > gpurun_out/pt_trace2_llm.txt 2>&1
PROBE_ONLY=c1 TSB_PT_TRACE=3 TSB_PT_PER_SM=4 timeout 200 python tools/pt_floor_probe.py 80 512 > gpurun_out/pt_trace2_c1.txt 2>&1
