timeout 600 python -m pytest -q -x tests/test_gpu_pipeline.py tests/test_gpu_crc_fused.py -p no:cacheprovider > gpurun_out/pack_tests.txt 2>&1
tail -1 gpurun_out/pack_tests.txt
for pk in 1 0 1 0; do TSB_PT_PACK=$pk PROBE_ONLY=c5llm timeout 200 python tools/pt_floor_probe.py 80 4096 | sed "s/}/, \"pack\": $pk}/"; done > gpurun_out/pack_ab.jsonl 2> gpurun_out/pack_ab.err
