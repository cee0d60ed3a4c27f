mkdir -p gpurun_out/p2
timeout 600 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_facade.py -x -q > gpurun_out/p2/pytest.log 2>&1
for st in 0 -1; do STRIDE=$st timeout 300 python tools/ring_overhead.py float32 > gpurun_out/p2/ring_s$st.txt 2>&1; done
timeout 900 python bench.py > gpurun_out/p2/bench.json 2> gpurun_out/p2/bench.err
