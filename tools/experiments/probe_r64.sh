mkdir -p gpurun_out/r64; o=gpurun_out/r64/res.txt
for cfg in 64:2:-1 32:2:2 32:3:-1 8:3:2; do
  IFS=: read r st res <<< "$cfg"
  for rep in 1 2; do
  if [ "$res" = "-1" ]; then unset TSB_CA_RESIDENT; else export TSB_CA_RESIDENT=$res; fi
  TSB_CA_R=$r TSB_CA_STAGES=$st timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r64/b.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/r64/b.json')); print('f32 R=$r st=$st res=$res', d['ms_per_step'], d['roofline']['frac'])" >> $o
  done
done
unset TSB_CA_RESIDENT
for cfg in 16:3 64:2 32:2 32:3; do
  IFS=: read r st <<< "$cfg"
  echo -n "u8 R=$r st=$st " >> $o
  TSB_CA_R=$r TSB_CA_STAGES=$st timeout 200 python tools/step_floor.py u8 host >> $o 2>&1
done
