mkdir -p gpurun_out/rr4
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/rr4/pytest.log 2>&1; echo rc=$? >> gpurun_out/rr4/pytest.log
for rep in 1 2 3; do timeout 300 python bench.py --no-cpu-baseline > gpurun_out/rr4/b$rep.json 2>/dev/null; done
timeout 600 python tools/bench_configs.py --only c2bf16,c4 > gpurun_out/rr4/cfg.jsonl 2>/dev/null
for k in u8 bf16 f32; do timeout 200 python tools/step_floor.py $k graph >> gpurun_out/rr4/floor.txt 2>&1; done
