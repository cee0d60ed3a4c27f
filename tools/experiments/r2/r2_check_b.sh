#!/bin/bash
out=gpurun_out/${1:-r2b}; mkdir -p $out
timeout 300 python tools/crc_bench.py 154.14272 77.07 38.5 9.633792 2.1 0.4 > $out/crc_tile.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize_configs.py tests/test_gpu_kernels.py -q -x -k "crc or fullsize or c4 or c5 or b256" > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:crc_tile -s 2 -c 1 \
    -o $out/full_crc_tile -f python tools/profile_one.py crc 4 > $out/ncu_crc.log 2>&1
