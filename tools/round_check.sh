#!/bin/bash
# usage (under gpurun): bash tools/round_check.sh <tag>
# what the driver runs at round end: the GPU suite, smoke(), the default bench
# and the reference arm.
tag=$1; out=gpurun_out/$tag; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -q -o faulthandler_timeout=300 > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $out/smoke.log 2>&1; echo "rc=$?" >> $out/smoke.log
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo "rc=$?" >> $out/bench.err
timeout 900 python bench.py --impl reference > $out/bench_ref.json 2> $out/bench_ref.err; echo "rc=$?" >> $out/bench_ref.err
# the one-GPU config table (per-batch and persistent passthrough) when asked
if [ -n "$CONFIGS" ]; then
  timeout 600 python tools/bench_configs.py --only c1,c5video,c5llm --slots 80 --steps 2048 > $out/configs.jsonl 2>> $out/configs.err
  timeout 600 python tools/bench_configs.py --only c1,c5video,c5llm --slots 80 --steps 2048 --persistent >> $out/configs.jsonl 2>> $out/configs.err
  timeout 600 python tools/bench_configs.py --only c2bf16,c4native,c4 --steps 512 >> $out/configs.jsonl 2>> $out/configs.err
fi
