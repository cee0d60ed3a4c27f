"""Sweep collate tuning knobs (TSB_CA_R, TSB_CA_STAGES); launches captured in a CUDA graph
so host overhead is excluded (device throughput only)."""
import os
import subprocess
import sys

code = r'''
import json, sys, torch
sys.path.insert(0, ".")
from paper_2409_18749_b200 import dataplane as dp
h, w, c, B, N = 224, 224, 3, int(sys.argv[1]), 16384
sb = h * w * c
store = torch.empty(N * sb, dtype=torch.uint8, device="cuda"); dp.make_store(store, 0, N, sb)
order = torch.from_numpy(dp.epoch_order(N, 0, 0)).cuda()
scale, bias = dp.norm_consts()
out = [torch.empty(B * c * h * w * 4, dtype=torch.uint8, device="cuda") for _ in range(3)]
res = {}
ITERS = 30
nb = N // B
for kind, name, ob in ((1, "f32", 4), (2, "bf16", 2), (0, "u8", 1)):
    def fn(i):
        j = i % nb
        dp.collate_augment(store, order[j * B:(j + 1) * B], B, h, w, c, 16, True, 0, 0, kind, out[i % 3], scale=scale, bias=bias)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for i in range(3): fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(ITERS): fn(i)
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / ITERS
    res[name] = [round(B * sb * (1 + ob) / ms / 1e6), round(ms * 1000, 1)]
print(json.dumps(res))
'''
B = sys.argv[3] if len(sys.argv) > 3 else "256"
for r in sys.argv[1].split(","):
    for st in sys.argv[2].split(","):
        env = dict(os.environ, TSB_CA_R=r, TSB_CA_STAGES=st)
        out = subprocess.run([sys.executable, "-c", code, B], env=env, capture_output=True, text=True)
        print(f"B={B} R={r} stages={st}: GB/s,us", out.stdout.strip() or out.stderr[-600:], flush=True)
