"""Quick device timing of the hot kernels (CUDA events, warm, inputs > L2)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2409_18749_b200 import dataplane as dp  # noqa: E402

torch.cuda.set_device(0)
h, w, c, B, N = 224, 224, 3, 256, 16384
sb = h * w * c
store = torch.empty(N * sb, dtype=torch.uint8, device="cuda")
dp.make_store(store, 0, N, sb)
order = dp.epoch_order(N, 0, 0)
didx_all = torch.from_numpy(order).cuda()
scale, bias = dp.norm_consts()
res = {}


def timeit(fn, iters=20):
    for _ in range(3):
        fn(0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(iters):
        fn(i)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


outs = {k: [torch.empty(B * c * h * w, dtype=dt, device="cuda") for _ in range(4)]
        for k, dt in ((1, torch.float32), (2, torch.bfloat16), (0, torch.uint8))}
for kind, name, ob in ((1, "f32", 4), (2, "bf16", 2), (0, "u8", 1)):
    def fn(i, kind=kind):
        bi = i % (N // B)
        dp.collate_augment(store, didx_all[bi * B:(bi + 1) * B], B, h, w, c, 16, True, 0, 0, kind,
                           outs[kind][i % 4], scale=scale, bias=bias)
    ms = timeit(fn)
    byts = B * sb * (1 + ob)
    res[f"collate_{name}"] = {"ms": ms, "GBps": byts / ms / 1e6, "Msamples_s": B / ms / 1e3}

gout = torch.empty(B * sb, dtype=torch.uint8, device="cuda")
ms = timeit(lambda i: dp.gather(store, didx_all[(i % 64) * B:((i % 64) + 1) * B], B, sb, gout))
res["gather_u8"] = {"ms": ms, "GBps": 2 * B * sb / ms / 1e6}
ms = timeit(lambda i: dp.fill_synthetic(gout, didx_all[(i % 64) * B:((i % 64) + 1) * B], B, 0, 0, sb))
res["fill_synthetic"] = {"ms": ms, "GBps": B * sb / ms / 1e6}
crc = torch.zeros(1, dtype=torch.int32, device="cuda")
big = outs[1][0]
ms = timeit(lambda i: dp.crc32(outs[1][i % 4], big.numel() * 4, crc))
res["crc32_f32slot"] = {"ms": ms, "GBps": big.numel() * 4 / ms / 1e6}
pinned = torch.empty(4096 * sb, dtype=torch.uint8).pin_memory()
ms = timeit(lambda i: dp.collate_augment(pinned, didx_all[0:B] % 4096, B, h, w, c, 16, True, 0, 0, 2,
                                          outs[2][0], scale=scale, bias=bias), iters=5)
res["collate_bf16_from_pinned"] = {"ms": ms, "pcie_GBps": B * sb / ms / 1e6}
src = outs[1][0]
dst = outs[1][1]
ms = timeit(lambda i: dst.copy_(src))
res["torch_copy_f32slot"] = {"ms": ms, "GBps": 2 * src.numel() * 4 / ms / 1e6}
ms = timeit(lambda i: dp.fanout(src, [dst], src.numel() * 4))
res["fanout_1dst"] = {"ms": ms, "GBps": 2 * src.numel() * 4 / ms / 1e6}
print(json.dumps(res, indent=1))
