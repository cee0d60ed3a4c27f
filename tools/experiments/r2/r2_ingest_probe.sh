#!/bin/bash
out=gpurun_out/${1:-ingp}; mkdir -p $out; shift
for n in ${@:-0 16 32 48 64}; do TSB_INGEST_CE=$n timeout 300 python tools/ingest_probe.py 96 | sed "s/^{/{\"ce_samples\": $n, /" >> $out/probe.jsonl 2>> $out/probe.err; done
timeout 300 python -m pytest tests/test_gpu_pipeline.py -q -x -k staged > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
