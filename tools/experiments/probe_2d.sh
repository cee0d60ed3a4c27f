mkdir -p gpurun_out/i2d; o=gpurun_out/i2d/res.txt
TSB_INGEST_2D=1 timeout 600 python -m pytest tests/test_gpu_pipeline.py -q -k staged > gpurun_out/i2d/pytest.log 2>&1; echo rc=$? >> gpurun_out/i2d/pytest.log
for mode in 0 1 0 1; do
  TSB_INGEST_2D=$mode timeout 300 python bench.py --no-cpu-baseline --steps 1024 > gpurun_out/i2d/b.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/i2d/b.json')); print('2d=$mode', d['e2e']['value'], d['e2e']['h2d_bytes_per_step'])" >> $o
done
