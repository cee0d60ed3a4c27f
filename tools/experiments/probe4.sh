mkdir -p gpurun_out/p4
for k in f32 bf16 u8; do
  for m in graph host device; do timeout 120 python tools/step_floor.py $k $m >> gpurun_out/p4/floor.txt 2>&1; done
  TSB_NO_PDL=1 timeout 120 python tools/step_floor.py $k host | sed 's/}/, "knob": "no_pdl"}/' >> gpurun_out/p4/floor.txt 2>&1
  TSB_NO_FUSED=1 timeout 120 python tools/step_floor.py $k host | sed 's/}/, "knob": "no_fused"}/' >> gpurun_out/p4/floor.txt 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/p4/launches_bf16_host.csv python tools/step_floor.py bf16 host > /dev/null 2>&1
