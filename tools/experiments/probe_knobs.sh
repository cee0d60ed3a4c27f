mkdir -p gpurun_out/knobs
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/knobs/pytest.log 2>&1; echo rc=$? >> gpurun_out/knobs/pytest.log
for m in host host1; do timeout 200 python tools/step_floor.py f32 $m >> gpurun_out/knobs/floor.txt 2>&1; done
