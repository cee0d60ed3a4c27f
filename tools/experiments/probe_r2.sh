mkdir -p gpurun_out/rr2; o=gpurun_out/rr2/res.txt
run() { # label, env...
  local label=$1; shift
  env "$@" timeout 300 python bench.py --no-cpu-baseline --steps 1024 > gpurun_out/rr2/b.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/rr2/b.json')); print('$label', d['ms_per_step'], d['roofline']['frac'])" >> $o
}
for r in 28 32 38 40 45 50; do
  for st in 2 3; do run "f32 R=$r st=$st" TSB_CA_R=$r TSB_CA_STAGES=$st; done
done
run "f32 R=45 st=2 res=2" TSB_CA_R=45 TSB_CA_STAGES=2 TSB_CA_RESIDENT=2
run "f32 R=45 st=2 res=4" TSB_CA_R=45 TSB_CA_STAGES=2 TSB_CA_RESIDENT=4
run "f32 R=45 st=2 blocked" TSB_CA_R=45 TSB_CA_STAGES=2 TSB_CA_ORDER=blocked
run "f32 R=45 st=2 nopdl" TSB_CA_R=45 TSB_CA_STAGES=2 TSB_NO_PDL=1
