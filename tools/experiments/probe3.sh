mkdir -p gpurun_out/p3
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/p3/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/p3/pytest.log
for g in 0 1; do GATE=$g timeout 300 python tools/ring_overhead.py float32 > gpurun_out/p3/ring_g$g.txt 2>&1; done
GATE=1 timeout 300 python tools/ring_overhead.py bfloat16 > gpurun_out/p3/ring_g1_bf16.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/p3/bench.json 2> gpurun_out/p3/bench.err
