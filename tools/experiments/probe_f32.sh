mkdir -p gpurun_out/f32
timeout 600 python -m pytest tests -m gpu -q -x -k "collate or augment or fullsize or pipeline or group" > gpurun_out/f32/pytest.log 2>&1; echo rc=$? >> gpurun_out/f32/pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/f32/bench.json 2> gpurun_out/f32/bench.err
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/f32/bench2.json 2>> gpurun_out/f32/bench.err
timeout 300 python tools/sweep_collate.py 8 3 > gpurun_out/f32/sweep.txt 2>&1
