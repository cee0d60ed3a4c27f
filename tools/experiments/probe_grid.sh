mkdir -p gpurun_out/grid; o=gpurun_out/grid/res.txt
run() { local label=$1; shift
  env "$@" timeout 300 python bench.py --no-cpu-baseline --steps 1024 > gpurun_out/grid/b.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/grid/b.json')); print('$label', d['ms_per_step'], d['roofline']['frac'])" >> $o; }
run "default"
run "grid=427" TSB_CA_GRID=427
run "grid=320" TSB_CA_GRID=320
run "grid=296" TSB_CA_GRID=296
run "grid=400" TSB_CA_GRID=400
run "R=38 grid=384" TSB_CA_R=38 TSB_CA_STAGES=2 TSB_CA_GRID=384
run "R=38 grid=439" TSB_CA_R=38 TSB_CA_STAGES=2 TSB_CA_GRID=439
run "R=56 grid=256" TSB_CA_R=56 TSB_CA_STAGES=2 TSB_CA_GRID=256
run "R=32 st2 (4/SM)" TSB_CA_R=32 TSB_CA_STAGES=2
run "R=32 grid=448" TSB_CA_R=32 TSB_CA_STAGES=2 TSB_CA_GRID=448
run "default again"
