mkdir -p gpurun_out/rr; o=gpurun_out/rr/res.txt
for r in 45 56 64 75 112; do
  for rep in 1 2; do
  TSB_CA_R=$r TSB_CA_STAGES=2 timeout 300 python bench.py --no-cpu-baseline > gpurun_out/rr/b.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/rr/b.json')); print('f32 R=$r st=2', d['ms_per_step'], d['roofline']['frac'])" >> $o
  done
done
for r in 56 64 75 112; do
  echo -n "bf16 R=$r st=2 " >> $o
  TSB_CA_R=$r TSB_CA_STAGES=2 timeout 300 python tools/bench_configs.py --only c2bf16 --steps 1024 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['us_per_batch'])" >> $o
done
for r in 56 64 112; do
  echo -n "u8 R=$r st=2 " >> $o
  TSB_CA_R=$r TSB_CA_STAGES=2 timeout 200 python tools/step_floor.py u8 host >> $o 2>&1
done
