mkdir -p gpurun_out/rr5; o=gpurun_out/rr5/res.txt
for rep in 1 2; do
for cfg in 45:2 38:2 56:2 64:2 32:2 45:3 75:2; do
  IFS=: read r st <<< "$cfg"
  TSB_CA_R=$r TSB_CA_STAGES=$st timeout 300 python bench.py --no-cpu-baseline --steps 1024 > gpurun_out/rr5/b.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/rr5/b.json')); print('f32 R=$r st=$st', d['ms_per_step'], d['roofline']['frac'])" >> $o
done
done
