#!/bin/bash
out=gpurun_out/quick_range; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_crc_fused.py tests/test_gpu_pipeline.py -q -p no:cacheprovider 2>&1 | tail -2 > $out/tests.txt
timeout 900 python bench.py --no-cpu-baseline > $out/bench.json 2> $out/bench.err
cat $out/tests.txt; python -c "
import json; d=json.load(open('$out/bench.json')); r=d['roofline']
print(d['value'], d['ms_per_step'], r['frac'], d['e2e']['value'], d['extra']['parity']['ok'], d['extra']['bf16']['avg_launch_ms'], d['clocks']['sm_mhz'])"
