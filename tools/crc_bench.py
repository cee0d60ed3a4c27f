"""Device CRC-32 throughput: python tools/crc_bench.py [MB ...]
(TSB_CRC_IMPL=v1 selects the round-1 kernel).  Prints one JSON line per size:
bytes / average launch time over 50 back-to-back launches (CUDA events),
checked against zlib on the host."""
import json
import os
import sys
import zlib

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_18749_b200 import dataplane as dp  # noqa: E402

sizes = [float(x) for x in sys.argv[1:]] or [154.14272, 77.07, 9.633792, 2.1]
torch.cuda.set_device(0)
for mb in sizes:
    n = int(mb * 1e6) // 16 * 16
    data = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda")
    out = torch.zeros(1, dtype=torch.int32, device="cuda")
    for _ in range(3):
        dp.crc32(data, n, out)
    torch.cuda.synchronize()
    # 50 calls captured in a CUDA graph: device time, not the Python launch loop
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(50):
                dp.crc32(data, n, out)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 50
    ok = (int(out.item()) & 0xFFFFFFFF) == zlib.crc32(data.cpu().numpy().tobytes())
    print(json.dumps({"impl": os.environ.get("TSB_CRC_IMPL", "tile"), "bytes": n,
                      "us": round(ms * 1e3, 2), "gbs": round(n / ms / 1e6, 1), "ok": ok}),
          flush=True)
