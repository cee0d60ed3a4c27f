mkdir -p gpurun_out/bf16; o=gpurun_out/bf16/res.txt
for cfg in 16:2:0 32:2:0 16:3:0 32:2:4 16:2:4 32:3:3 64:2:2 8:3:0; do
  IFS=: read r st res <<< "$cfg"
  for rep in 1 2; do
  echo -n "R=$r st=$st resident=$res " >> $o
  TSB_CA_R=$r TSB_CA_STAGES=$st TSB_CA_RESIDENT=$res timeout 300 python tools/bench_configs.py --only c2bf16 --steps 1024 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['us_per_batch'])" >> $o
  done
done
