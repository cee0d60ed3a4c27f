for ep in 8 1; do TSB_EPOCHS_PER_LAUNCH=$ep TSB_PT_PER_SM=4 timeout 200 python tools/pt_floor_probe.py 80 2048 | sed "s/}/, \"epl\": $ep}/"; done > gpurun_out/pt_v5.jsonl 2> gpurun_out/pt_v5.err
timeout 300 python tools/bench_configs.py --only c1,c5video,c5llm --slots 80 --steps 2048 > gpurun_out/pt_v5_perbatch.jsonl 2>> gpurun_out/pt_v5.err
for w in 0 300; do TSB_FR_CHECKSUM=1 TSB_FR_WORK_US=$w timeout 300 python tools/facade_rate.py 2000 >> gpurun_out/facade_bound.jsonl 2>> gpurun_out/pt_v5.err; done
