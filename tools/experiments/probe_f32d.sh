mkdir -p gpurun_out/f32d
o=gpurun_out/f32d/res.txt
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/f32d/pytest.log 2>&1; echo rc=$? >> gpurun_out/f32d/pytest.log
for rep in 1 2 3; do
  timeout 300 python bench.py --no-cpu-baseline > gpurun_out/f32d/b$rep.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/f32d/b$rep.json')); print('default', d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'])" >> $o
done
for res in 0 2 3; do for r in 16 32; do
  echo -n "bf16 R=$r resident=$res " >> $o
  TSB_CA_R=$r TSB_CA_RESIDENT=$res timeout 300 python tools/bench_configs.py --only c2bf16 --steps 1024 >> $o 2>/dev/null
done; done
