mkdir -p gpurun_out/thr5; o=gpurun_out/thr5/res.txt
P=paper_2409_18749_b200
for t in 256 128 256 128; do
  cp $P/libtsb200_b$t.so $P/libtsb200.so; touch $P/libtsb200.so
  echo -n "bf16 threads=$t " >> $o
  timeout 300 python tools/bench_configs.py --only c2bf16 --steps 1024 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['us_per_batch'])" >> $o
  echo -n "u8 threads=$t " >> $o
  timeout 200 python tools/step_floor.py u8 host 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['us_per_batch'])" >> $o
done
cp $P/libtsb200_b256.so $P/libtsb200.so
