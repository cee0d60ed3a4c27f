mkdir -p gpurun_out/bfma; o=gpurun_out/bfma/res.txt
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/bfma/pytest.log 2>&1; echo rc=$? >> gpurun_out/bfma/pytest.log
for fm in 1 0 1 0; do
  echo -n "bf16 fma=$fm " >> $o
  TSB_BF16_FMA=$fm timeout 300 python tools/bench_configs.py --only c2bf16 --steps 1024 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['us_per_batch'], d['value'])" >> $o
done
