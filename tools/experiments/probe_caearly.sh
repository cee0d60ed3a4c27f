mkdir -p gpurun_out/caearly; o=gpurun_out/caearly/res.txt
for e in 0 1 0 1; do
  TSB_CA_EARLY=$e timeout 300 python bench.py --no-cpu-baseline --steps 1024 > gpurun_out/caearly/b.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/caearly/b.json')); print('f32 early=$e', d['ms_per_step'], d['roofline']['frac'])" >> $o
  echo -n "bf16 early=$e " >> $o
  TSB_CA_EARLY=$e timeout 300 python tools/bench_configs.py --only c2bf16 --steps 1024 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['us_per_batch'])" >> $o
done
