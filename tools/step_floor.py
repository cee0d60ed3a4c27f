"""Where does a producer step go?  Per-batch device time of the native loop
(tsb_produce_range) vs the bare collate kernel in a CUDA graph, per output
kind.  Knobs (env, read once): TSB_NO_PDL, TSB_NO_FUSED.
usage: python tools/step_floor.py <f32|bf16|u8> <mode>  mode: graph|host|host1|device
(host1: one batch per tsb_produce_range call, the facade's pattern)"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2409_18749_b200 import AugmentSpec, CollateLoader, DatasetSpec, StoreSource  # noqa: E402
from paper_2409_18749_b200._lib import GATE_DEVICE, GATE_HOST  # noqa: E402
from paper_2409_18749_b200.ring import DeviceRing, produce_range  # noqa: E402

kind, mode = sys.argv[1], sys.argv[2]
B, N, K = 256, 16384, 256
torch.cuda.set_device(0)
store = StoreSource.synthetic(0, N, (224, 224, 3))
dt = {"f32": "float32", "bf16": "bfloat16", "u8": "uint8"}[kind]
ld = CollateLoader(DatasetSpec(store, N, B), AugmentSpec(out_dtype=dt))
L = len(ld)
s = torch.cuda.Stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
if mode == "graph":
    outs = [torch.empty(ld.batch_nbytes, dtype=torch.uint8, device="cuda") for _ in range(8)]
    with torch.cuda.stream(s):
        for i in range(3):
            ld.produce_into(outs[i].data_ptr(), 0, i, s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(32):
            ld.produce_into(outs[i % 8].data_ptr(), 0, i % L, s)
    g.replay()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(K // 32):
        g.replay()
    e1.record()
else:
    ring = DeviceRing(8, ld.batch_nbytes, 1, control="device" if mode == "device" else "host")

    per_call = 1 if mode == "host1" else 1 << 30

    def run(q0, n):
        q = q0
        while q < q0 + n:
            ep, bi = divmod(q - 1, L)
            m = min(q0 + n - q, L - bi, per_call)
            a = ld.produce_args(ep)
            a.gate = GATE_DEVICE if mode == "device" else GATE_HOST
            produce_range(ring, a, q, bi, m, [], stream=s)
            q += m

    import time as _t

    run(1, 16)
    s.synchronize()
    e0.record(s)
    h0 = _t.perf_counter()
    run(17, K)
    host_us = (_t.perf_counter() - h0) * 1e6 / K
    e1.record(s)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / K
print(json.dumps({"kind": kind, "mode": mode, "us_per_batch": round(ms * 1000, 2),
                  "host_enqueue_us_per_batch": round(host_us, 2) if mode != "graph" else None,
                  "Msamples_s": round(B / ms / 1e3, 3)}))
