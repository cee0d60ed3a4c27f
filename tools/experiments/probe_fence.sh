mkdir -p gpurun_out/fence; o=gpurun_out/fence/res.txt
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/fence/pytest.log 2>&1; echo rc=$? >> gpurun_out/fence/pytest.log
for fa in 0 1 0 1; do
  TSB_FENCE_ALL=$fa timeout 300 python tools/bench_configs.py --only c1,c5video,c5llm --steps 1024 2>/dev/null | python -c "
import json,sys
for l in sys.stdin: d=json.loads(l); print('fence_all=$fa', d['config'][:12], d['us_per_batch'])" >> $o
  TSB_FENCE_ALL=$fa timeout 300 python bench.py --no-cpu-baseline --steps 1024 > gpurun_out/fence/b.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/fence/b.json')); print('fence_all=$fa C2 f32', d['ms_per_step'], d['roofline']['frac'])" >> $o
done
