mkdir -p gpurun_out/rr6; o=gpurun_out/rr6/res.txt
for rep in 1 2; do
for cfg in 32:2 28:2 45:2 25:2; do
  IFS=: read r st <<< "$cfg"
  TSB_CA_R=$r TSB_CA_STAGES=$st timeout 300 python bench.py --no-cpu-baseline --steps 1024 > gpurun_out/rr6/b.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/rr6/b.json')); print('f32 R=$r st=$st', d['ms_per_step'], d['roofline']['frac'])" >> $o
  echo -n "bf16 R=$r st=$st " >> $o
  TSB_CA_R=$r TSB_CA_STAGES=$st timeout 300 python tools/bench_configs.py --only c2bf16 --steps 1024 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['us_per_batch'])" >> $o
  echo -n "u8 R=$r st=$st " >> $o
  TSB_CA_R=$r TSB_CA_STAGES=$st timeout 200 python tools/step_floor.py u8 host 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['us_per_batch'])" >> $o
done
done
