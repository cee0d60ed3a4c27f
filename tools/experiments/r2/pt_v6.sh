for p in 2 4 8; do TSB_PT_PER_SM=$p timeout 200 python tools/pt_floor_probe.py 80 2048; done > gpurun_out/pt_v6.jsonl 2> gpurun_out/pt_v6.err
TSB_EPOCHS_PER_LAUNCH=8 TSB_PT_PER_SM=4 timeout 200 python tools/pt_floor_probe.py 80 2048 | sed 's/}/, "epl": 8}/' >> gpurun_out/pt_v6.jsonl 2>> gpurun_out/pt_v6.err
TSB_FR_CHECKSUM=1 timeout 300 python tools/facade_rate.py 4000 >> gpurun_out/pt_v6_facade.jsonl 2>> gpurun_out/pt_v6.err
timeout 600 python -m pytest -q -x tests/test_gpu_pipeline.py tests/test_gpu_crc_fused.py > gpurun_out/pt_v6_tests.txt 2>&1
