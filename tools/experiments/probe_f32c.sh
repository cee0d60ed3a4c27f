mkdir -p gpurun_out/f32c
o=gpurun_out/f32c/res.txt
for cfg in "4:0:0:0" "8:0:2:0" "8:0:3:0" "4:0:3:0" "8:0:2:1" "16:0:2:0" "8:2:0:0"; do
  IFS=: read r occ res nopdl <<< "$cfg"
  for rep in 1 2; do
  TSB_CA_R=$r TSB_CA_OCC=$occ TSB_CA_RESIDENT=$res TSB_NO_PDL=$nopdl timeout 300 python bench.py --no-cpu-baseline > gpurun_out/f32c/b.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/f32c/b.json')); print('R=$r occ=$occ resident=$res nopdl=$nopdl', d['ms_per_step'], d['roofline']['frac'])" >> $o
  done
done
