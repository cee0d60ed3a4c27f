PROBE_ONLY=c1 TSB_PT_TRACE=3 timeout 200 python tools/pt_floor_probe.py 80 512 > gpurun_out/pt_trace3_c1.txt 2>&1
PROBE_BOTH=1 PROBE_ONLY=c1 TSB_PT_TRACE=3 timeout 200 python tools/pt_floor_probe.py 80 512 > gpurun_out/pt_trace3_c1_both.txt 2>&1
