#!/bin/bash
out=gpurun_out/${1:-ingp}; mkdir -p $out
for c in 8192 16384 32768 65536 150528; do TSB_IG_CHUNK=$c timeout 300 python tools/ingest_probe.py 96 >> $out/probe.jsonl 2>> $out/probe.err; done
timeout 300 python tools/h2d_probe.py > $out/h2d.json 2>> $out/probe.err
