"""PCIe ingest probe: pinned-host -> HBM by the copy engine (one contiguous
copy; 256 scattered 150 KB samples via per-sample memcpy), and by the collate
kernel reading pinned memory directly."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2409_18749_b200 import dataplane as dp  # noqa: E402

torch.cuda.set_device(0)
B, SB, N = 256, 150528, 4096
host = torch.empty(N * SB, dtype=torch.uint8).pin_memory()
host.random_(0, 255)
dev = torch.empty(B * SB, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
res = {}


def timeit(fn, iters=20):
    with torch.cuda.stream(s):
        fn()
        s.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(iters):
            fn()
        e1.record(s)
        s.synchronize()
    return e0.elapsed_time(e1) / iters


ms = timeit(lambda: dev.copy_(host[:B * SB], non_blocking=True))
res["h2d_contiguous_38MB_GBps"] = round(B * SB / ms / 1e6, 1)
idx = torch.randperm(N)[:B].tolist()


def scattered():
    for j, i in enumerate(idx):
        dev[j * SB:(j + 1) * SB].copy_(host[i * SB:(i + 1) * SB], non_blocking=True)


ms = timeit(scattered, iters=5)
res["h2d_256_scattered_copies_GBps"] = round(B * SB / ms / 1e6, 1)
t0 = time.perf_counter()
scattered()
res["host_enqueue_256_copies_ms"] = round((time.perf_counter() - t0) * 1e3, 3)
didx = torch.tensor(idx, dtype=torch.int64, device="cuda")
out = torch.empty(B * 3 * 224 * 224 * 4, dtype=torch.uint8, device="cuda")
scale, bias = dp.norm_consts()
ms = timeit(lambda: dp.collate_augment(host, didx, B, 224, 224, 3, 16, True, 0, 0, 1, out,
                                       scale=scale, bias=bias, stream=s), iters=5)
res["collate_f32_direct_from_pinned_GBps"] = round(B * SB / ms / 1e6, 1)
ms = timeit(lambda: dp.gather(host, didx, B, SB, dev, stream=s), iters=5)
res["gather_direct_from_pinned_GBps"] = round(B * SB / ms / 1e6, 1)
print(json.dumps(res, indent=1))
