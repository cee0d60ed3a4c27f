#!/bin/bash
out=gpurun_out/${1:-crcab}; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -k crc > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
for k in 2 3 4; do
  TSB_CRC_CHAINS=$k timeout 300 python tools/crc_bench.py 154.14272 38.5 9.633792 2.1 0.4 > $out/crc_k$k.jsonl 2>&1
done
TSB_CRC_CHAINS=3 timeout 600 python -m pytest tests/test_gpu_kernels.py -q -k crc > $out/pytest_k3.log 2>&1; echo "rc=$?" >> $out/pytest_k3.log
TSB_CRC_CHAINS=4 timeout 600 python -m pytest tests/test_gpu_kernels.py -q -k crc > $out/pytest_k4.log 2>&1; echo "rc=$?" >> $out/pytest_k4.log
