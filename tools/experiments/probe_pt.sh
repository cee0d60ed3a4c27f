mkdir -p gpurun_out/pt2
for ps in 2 8; do
  TSB_PT_PER_SM=$ps timeout 300 python tools/bench_configs.py --only c1,c5video,c5llm --steps 2048 | sed "s/}/, \"per_sm\": $ps, \"persistent\": false}/" >> gpurun_out/pt2/cfg.jsonl 2>/dev/null
  TSB_PT_PER_SM=$ps timeout 300 python tools/bench_configs.py --only c1,c5video,c5llm --steps 2048 --persistent | sed "s/}/, \"per_sm\": $ps, \"persistent\": true}/" >> gpurun_out/pt2/cfg.jsonl 2>/dev/null
done
timeout 300 python bench.py --no-cpu-baseline --steps 1024 > gpurun_out/pt2/bench.json 2>/dev/null
