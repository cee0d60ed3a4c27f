#!/bin/bash
out=gpurun_out/${1:-rb}; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_facade_multi.py tests/test_gpu_fullsize_configs.py tests/test_gpu_kernels.py -q -x -o faulthandler_timeout=300 > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
bash tools/experiments/r2/r2_ncu.sh ${1:-rb}/ncu rebatch
