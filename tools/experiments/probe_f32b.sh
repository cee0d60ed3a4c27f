mkdir -p gpurun_out/f32b
o=gpurun_out/f32b/res.txt
for cfg in "4:0:0" "8:2:0" "8:2:1" "8:3:0" "8:0:0" "4:2:0" "16:2:0"; do
  IFS=: read r occ nopdl <<< "$cfg"
  for rep in 1 2; do
  TSB_CA_R=$r TSB_CA_OCC=$occ TSB_NO_PDL=$nopdl timeout 300 python bench.py --no-cpu-baseline > gpurun_out/f32b/b.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/f32b/b.json')); print('R=$r occ=$occ nopdl=$nopdl', d['ms_per_step'], d['roofline']['frac'])" >> $o
  done
done
