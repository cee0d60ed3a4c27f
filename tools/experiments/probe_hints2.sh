mkdir -p gpurun_out/h2; o=gpurun_out/h2/res.txt
run() { local label=$1; shift
  env "$@" timeout 300 python bench.py --no-cpu-baseline --steps 1024 > gpurun_out/h2/b.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/h2/b.json')); print('$label', d['ms_per_step'], d['roofline']['frac'])" >> $o; }
for rep in 1 2; do
run "default"
run "ldhint=0" TSB_CA_LDHINT=0
run "st=plain" TSB_CA_ST=plain
run "both off" TSB_CA_LDHINT=0 TSB_CA_ST=plain
run "direct" TSB_CA_IMPL=direct
done
