mkdir -p gpurun_out/p6
timeout 900 python -m pytest tests/test_gpu_facade_multi.py -x -q > gpurun_out/p6/pytest_multi.log 2>&1; echo "rc=$?" >> gpurun_out/p6/pytest_multi.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/p6/pytest_all.log 2>&1; echo "rc=$?" >> gpurun_out/p6/pytest_all.log
