#!/bin/bash
# pinned-store ingest: host-packed rows + one copy per batch vs the gather kernel
out=gpurun_out/${1:-hp}; mkdir -p $out
nproc > $out/nproc.txt
TSB_INGEST=hostpack timeout 300 python -m pytest tests/test_gpu_pipeline.py -q -x -k staged > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
timeout 300 python tools/ingest_probe.py 96 | sed 's/^{/{"mode": "gather", /' >> $out/probe.jsonl 2>> $out/probe.err
for t in 4 7 12; do TSB_INGEST=hostpack TSB_INGEST_THREADS=$t timeout 300 python tools/ingest_probe.py 96 | sed "s/^{/{\"mode\": \"hostpack\", \"threads\": $t, /" >> $out/probe.jsonl 2>> $out/probe.err; done
TSB_INGEST=hostpack timeout 600 python bench.py --no-cpu-baseline --steps 64 > $out/bench_hostpack.json 2> $out/bench_hostpack.err
