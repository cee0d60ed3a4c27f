#!/bin/bash
# One GPU session: tests, smoke, bench, ncu launch list + full capture of the collate kernel.
# usage (under gpurun): bash tools/gpu_round.sh [tag]
tag=${1:-r1}
out=gpurun_out/$tag
mkdir -p "$out"
nvidia-smi > "$out/nvidia-smi.txt" 2>&1
nproc > "$out/nproc.txt"; grep -m1 "model name" /proc/cpuinfo >> "$out/nproc.txt"
timeout 900 python -m pytest tests -m gpu -x -q > "$out/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$out/pytest_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$out/smoke.log" 2>&1; echo "smoke rc=$?" >> "$out/smoke.log"
timeout 900 python bench.py > "$out/bench.json" 2> "$out/bench.err"; echo "bench rc=$?" >> "$out/bench.err"
timeout 600 python bench.py --impl reference --steps 8 --warmup 3 > "$out/bench_ref.json" 2> "$out/bench_ref.err"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$out/launches.csv" \
    python bench.py --steps 4 --warmup 3 --no-cpu-baseline > "$out/bench_under_ncu.log" 2>&1
for k in f32 bf16 u8 crc; do
  timeout 600 ncu --set full --clock-control none --import-source on -s 2 -c 1 \
      -o "$out/prof_$k" -f python tools/profile_one.py $k 4 > "$out/prof_$k.log" 2>&1
done
echo done > "$out/DONE"
