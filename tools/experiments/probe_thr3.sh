mkdir -p gpurun_out/thr3
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/thr3/pytest.log 2>&1; echo rc=$? >> gpurun_out/thr3/pytest.log
for rep in 1 2; do timeout 300 python bench.py --no-cpu-baseline > gpurun_out/thr3/b$rep.json 2>/dev/null; done
timeout 300 python tools/bench_configs.py --only c2bf16 > gpurun_out/thr3/cfg.jsonl 2>/dev/null
