mkdir -p gpurun_out/early; o=gpurun_out/early/res.txt
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_kernels.py tests/test_gpu_facade.py tests/test_gpu_group.py -q -x > gpurun_out/early/pytest.log 2>&1; echo rc=$? >> gpurun_out/early/pytest.log
for e in 1 0 1 0; do
  TSB_PT_EARLY=$e timeout 300 python tools/bench_configs.py --only c1,c5video,c5llm --steps 2048 2>/dev/null | python -c "
import json,sys
for l in sys.stdin: d=json.loads(l); print('early=$e', d['config'][:12], d['us_per_batch'], d['value'])" >> $o
done
