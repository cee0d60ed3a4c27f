#!/bin/bash
out=gpurun_out/${1:-facade}; mkdir -p $out
timeout 300 python tools/facade_rate.py 4000 > $out/fr_nocrc.json 2> $out/fr_nocrc.err
TSB_FR_CHECKSUM=1 timeout 300 python tools/facade_rate.py 4000 > $out/fr_crc.json 2> $out/fr_crc.err
TSB_PROFILE_PRODUCER=$out/prof_producer.txt timeout 300 python tools/facade_rate.py 4000 > $out/fr_prof.json 2>&1
TSB_PROFILE_CONSUMER=$out/prof_consumer.txt timeout 300 python tools/facade_rate.py 4000 > $out/fr_profc.json 2>&1
