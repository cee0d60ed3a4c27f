#!/bin/bash
# e2e A/B of the pinned-store ingest: gather kernel (default) vs direct TMA from the pinned store
out=gpurun_out/${1:-ingab}; mkdir -p $out; shift
TSB_INGEST=direct timeout 300 python -m pytest tests/test_gpu_pipeline.py -q -x -k "staged" > $out/pytest_direct.log 2>&1; echo "rc=$?" >> $out/pytest_direct.log
for m in ${@:-gather direct}; do
  if [ $m != gather ]; then export TSB_INGEST=$m; else unset TSB_INGEST; fi
  timeout 600 python bench.py --no-cpu-baseline --steps 64 > $out/bench_$m.json 2> $out/bench_$m.err
done
