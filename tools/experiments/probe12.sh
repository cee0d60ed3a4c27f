mkdir -p gpurun_out/p12
timeout 300 python tools/h2d_probe.py > gpurun_out/p12/h2d.json 2>&1
timeout 600 python tools/sweep_collate.py 4,8,16,32 2,3,4 > gpurun_out/p12/sweep.txt 2>&1
