mkdir -p gpurun_out/thr; o=gpurun_out/thr/res.txt
P=paper_2409_18749_b200
for t in 256 128 384 512; do
  cp $P/libtsb200_t$t.so $P/libtsb200.so; touch $P/libtsb200.so
  for rep in 1 2; do
    timeout 300 python bench.py --no-cpu-baseline --steps 1024 > gpurun_out/thr/b.json 2>gpurun_out/thr/err.txt
    python -c "import json; d=json.load(open('gpurun_out/thr/b.json')); print('f32 threads=$t', d['ms_per_step'], d['roofline']['frac'])" >> $o 2>>gpurun_out/thr/err.txt
  done
  echo -n "bf16 threads=$t " >> $o
  timeout 300 python tools/bench_configs.py --only c2bf16 --steps 1024 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['us_per_batch'])" >> $o
done
cp $P/libtsb200_t256.so $P/libtsb200.so
