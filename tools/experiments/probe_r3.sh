mkdir -p gpurun_out/rr3; o=gpurun_out/rr3/res.txt
for cfg in 45:2 45:3 38:2 64:2 75:3 32:2; do
  IFS=: read r st <<< "$cfg"
  echo -n "bf16 R=$r st=$st " >> $o
  TSB_CA_R=$r TSB_CA_STAGES=$st timeout 300 python tools/bench_configs.py --only c2bf16 --steps 1024 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['us_per_batch'])" >> $o
done
for cfg in 45:2 45:3 32:2 38:3 75:2; do
  IFS=: read r st <<< "$cfg"
  echo -n "u8 R=$r st=$st " >> $o
  TSB_CA_R=$r TSB_CA_STAGES=$st timeout 200 python tools/step_floor.py u8 host >> $o 2>&1
done
