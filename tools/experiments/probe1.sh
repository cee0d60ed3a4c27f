mkdir -p gpurun_out/p1
python tools/membw_ref.py > gpurun_out/p1/membw.json 2>&1
python tools/quick_timing.py > gpurun_out/p1/quick.json 2>&1
for st in 1 2 4; do STRIDE=$st python tools/ring_overhead.py float32 > gpurun_out/p1/ring_s$st.txt 2>&1; done
SLOTS=16 STRIDE=4 python tools/ring_overhead.py float32 > gpurun_out/p1/ring_16_s4.txt 2>&1
python tools/sweep_collate.py 2,4,8 3,4,6 > gpurun_out/p1/sweep.txt 2>&1
./tools/bw_probe > gpurun_out/p1/bw_probe.txt 2>&1
