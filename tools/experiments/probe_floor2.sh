mkdir -p gpurun_out/floor2; o=gpurun_out/floor2/floor.txt
for m in graph host host1; do timeout 200 python tools/step_floor.py f32 $m >> $o 2>&1; done
TSB_NO_PDL=1 timeout 200 python tools/step_floor.py f32 host >> $o 2>&1
timeout 200 python tools/sweep_collate.py 8 3 >> $o 2>&1
