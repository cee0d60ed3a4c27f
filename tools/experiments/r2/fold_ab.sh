for f in 1 2 3; do TSB_CC_FOLD=$f timeout 600 python -m pytest -q -x tests/test_gpu_crc_fused.py -p no:cacheprovider 2>&1 | tail -1 | sed "s/^/fold $f: /"; done > gpurun_out/fold_tests.txt
for f in 0 1 2 3 0 1 2 3; do TSB_CC_FOLD=$f TIMING_PERSIST=1 timeout 300 python tools/crc_fused_timing.py f32,bf16,u8 512 2>/dev/null | grep '"checksum": true' | sed "s/}/, \"fold\": $f}/"; done > gpurun_out/fold_ab.jsonl
cat gpurun_out/fold_tests.txt
