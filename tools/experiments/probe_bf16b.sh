mkdir -p gpurun_out/bf16b; o=gpurun_out/bf16b/res.txt
for cfg in 64:2:2 64:3:1 32:4:2 32:2:2 64:2:0 32:3:2 64:1:2; do
  IFS=: read r st res <<< "$cfg"
  for rep in 1 2; do
  echo -n "R=$r st=$st resident=$res " >> $o
  TSB_CA_R=$r TSB_CA_STAGES=$st TSB_CA_RESIDENT=$res timeout 300 python tools/bench_configs.py --only c2bf16 --steps 1024 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['us_per_batch'])" >> $o
  done
done
