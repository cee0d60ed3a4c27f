#!/bin/bash
out=gpurun_out/${1:-facade}; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_control.py tests/test_gpu_facade.py tests/test_gpu_facade_multi.py tests/test_gpu_fullsize_configs.py -q -x > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
timeout 300 python tools/facade_rate.py 4000 > $out/fr_nocrc.json 2> $out/fr_nocrc.err
TSB_FR_CHECKSUM=1 timeout 300 python tools/facade_rate.py 4000 > $out/fr_crc.json 2> $out/fr_crc.err
TSB_FR_DEPTH=2 timeout 300 python tools/facade_rate.py 4000 > $out/fr_d2.json 2> $out/fr_d2.err
TSB_PROFILE_PRODUCER=$out/prof_producer.txt timeout 300 python tools/facade_rate.py 4000 > $out/fr_prof.json 2>&1
