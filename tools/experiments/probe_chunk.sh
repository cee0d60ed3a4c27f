mkdir -p gpurun_out/chunk; o=gpurun_out/chunk/res.txt
P=paper_2409_18749_b200
for c in 16384 8192 4096 32768 16384 8192 4096 32768; do
  cp $P/libtsb200_c$c.so $P/libtsb200.so; touch $P/libtsb200.so
  timeout 300 python tools/bench_configs.py --only c1,c5video,c5llm --steps 2048 2>/dev/null | python -c "
import json,sys
for l in sys.stdin: d=json.loads(l); print('chunk=$c', d['config'][:12], d['us_per_batch'])" >> $o
done
cp $P/libtsb200_c16384.so $P/libtsb200.so
