mkdir -p gpurun_out/thr4; o=gpurun_out/thr4/res.txt
P=paper_2409_18749_b200
for t in 128 96 192 128 96 192; do
  cp $P/libtsb200_f$t.so $P/libtsb200.so; touch $P/libtsb200.so
  timeout 300 python bench.py --no-cpu-baseline --steps 1024 > gpurun_out/thr4/b.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/thr4/b.json')); print('f32 threads=$t', d['ms_per_step'], d['roofline']['frac'])" >> $o
done
cp $P/libtsb200_f128.so $P/libtsb200.so
