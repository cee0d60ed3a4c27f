#!/bin/bash
# usage (under gpurun): bash tools/gpu_check.sh <tag> [bench args...]
tag=$1; shift
out=gpurun_out/$tag; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -q -o faulthandler_timeout=300 > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
timeout 900 python bench.py "$@" > $out/bench.json 2> $out/bench.err; echo "rc=$?" >> $out/bench.err
