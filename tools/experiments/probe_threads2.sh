mkdir -p gpurun_out/thr2; o=gpurun_out/thr2/res.txt
P=paper_2409_18749_b200
cp $P/libtsb200_t128.so $P/libtsb200.so; touch $P/libtsb200.so
for cfg in 32:2 38:2 45:2 56:2 64:2 45:3 75:2; do
  IFS=: read r st <<< "$cfg"
  TSB_CA_R=$r TSB_CA_STAGES=$st timeout 300 python bench.py --no-cpu-baseline --steps 1024 > gpurun_out/thr2/b.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/thr2/b.json')); print('f32 t128 R=$r st=$st', d['ms_per_step'], d['roofline']['frac'])" >> $o
done
cp $P/libtsb200_t256.so $P/libtsb200.so
