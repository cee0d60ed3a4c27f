#!/bin/bash
# fused collate+CRC: parity tests, the ingest tests, bench lines (checksum on/off), ncu of the fused kernel
out=gpurun_out/${1:-crcf}; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_crc_fused.py -q -o faulthandler_timeout=240 > $out/pytest_crc.log 2>&1; echo "rc=$?" >> $out/pytest_crc.log
timeout 600 python -m pytest tests/test_gpu_pipeline.py -q -k "staged or ingest" -o faulthandler_timeout=240 > $out/pytest_ingest.log 2>&1; echo "rc=$?" >> $out/pytest_ingest.log
timeout 600 python bench.py --no-cpu-baseline > $out/bench.json 2> $out/bench.err; echo "rc=$?" >> $out/bench.err
timeout 600 python bench.py --no-cpu-baseline --checksum off > $out/bench_nocrc.json 2> $out/bench_nocrc.err; echo "rc=$?" >> $out/bench_nocrc.err
bash tools/experiments/r2/r2_ncu.sh ${1:-crcf}/ncu f32crc
