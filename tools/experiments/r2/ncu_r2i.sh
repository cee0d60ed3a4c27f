python tools/profile_r2.py ingest 4 && python tools/profile_r2.py llm_persistent 64 || exit 1
ncu --set full --clock-control none --import-source on -k regex:ingest_gather -s 2 -c 1 -o gpurun_out/ncu_ingest python tools/profile_r2.py ingest 4 > gpurun_out/ncu_ingest.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:persistent_passthrough -c 1 -o gpurun_out/ncu_llm_persistent python tools/profile_r2.py llm_persistent 64 > gpurun_out/ncu_llm_persistent.log 2>&1
ls gpurun_out/*.ncu-rep
