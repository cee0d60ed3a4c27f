mkdir -p gpurun_out/pers; o=gpurun_out/pers/res.txt
timeout 600 python -m pytest tests/test_gpu_pipeline.py -q -x -k persistent > gpurun_out/pers/pytest.log 2>&1; echo rc=$? >> gpurun_out/pers/pytest.log
for rep in 1 2; do
  timeout 300 python tools/bench_configs.py --only c1,c5video,c5llm --steps 2048 --persistent 2>/dev/null | python -c "
import json,sys
for l in sys.stdin: d=json.loads(l); print('persistent', d['config'][:12], d['us_per_batch'], d['value'])" >> $o
  timeout 300 python tools/bench_configs.py --only c1,c5video,c5llm --steps 2048 2>/dev/null | python -c "
import json,sys
for l in sys.stdin: d=json.loads(l); print('per-launch', d['config'][:12], d['us_per_batch'], d['value'])" >> $o
done
