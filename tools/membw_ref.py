"""Reference HBM bandwidth for the traffic mixes the hot kernels see (torch kernels)."""
import json
import torch

torch.cuda.set_device(0)
res = {}


def t(fn, nbytes, iters=30):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / iters
    return round(nbytes / ms / 1e6)


N = 38535168  # one batch of u8 224x224x3 x256
src = torch.empty(N, dtype=torch.uint8, device="cuda").random_(0, 255)
dst4 = torch.empty(4 * N, dtype=torch.uint8, device="cuda")
dst2 = torch.empty(2 * N, dtype=torch.uint8, device="cuda")
big = torch.empty(8 * N, dtype=torch.uint8, device="cuda")
res["write_only_154MB"] = t(lambda: dst4.fill_(7), 4 * N)
res["copy_1to1_154MB"] = t(lambda: dst4[:4 * N // 2].copy_(big[:2 * N]), 4 * N)
res["read1_write4_192MB"] = t(lambda: dst4.view(4, N).copy_(src.expand(4, N)), 5 * N)
res["read1_write2_115MB"] = t(lambda: dst2.view(2, N).copy_(src.expand(2, N)), 3 * N)
res["copy_1to1_77MB"] = t(lambda: dst2[:N].copy_(big[:N]), 2 * N)
print(json.dumps(res, indent=1))
