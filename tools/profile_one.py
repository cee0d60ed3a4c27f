"""Launch one hot kernel a few times (for ncu): python tools/profile_one.py <what> [iters]."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2409_18749_b200 import dataplane as dp  # noqa: E402

what = sys.argv[1]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
torch.cuda.set_device(0)
h, w, c, B, N = 224, 224, 3, 256, 16384
sb = h * w * c
store = torch.empty(N * sb, dtype=torch.uint8, device="cuda")
dp.make_store(store, 0, N, sb)
order = torch.from_numpy(dp.epoch_order(N, 0, 0)).cuda()
scale, bias = dp.norm_consts()
kind = {"f32": 1, "bf16": 2, "u8": 0}
out = torch.empty(B * c * h * w * 4, dtype=torch.uint8, device="cuda")
crc = torch.zeros(1, dtype=torch.int32, device="cuda")
out2 = torch.empty(B * c * h * w * 2, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize()
for i in range(iters):
    idx = order[(i % 64) * B:((i % 64) + 1) * B]
    if what in kind:
        dp.collate_augment(store, idx, B, h, w, c, 16, True, 0, 0, kind[what], out, scale=scale,
                           bias=bias)
    elif what == "crc":
        dp.crc32(out, B * c * h * w * 4, crc)
    elif what == "gather":
        dp.gather(store, idx, B, sb, out)
    elif what == "fanout2_bf16":  # collate MULTI: one pass into two destination slots
        dp.collate_augment_fanout(store, idx, B, h, w, c, 16, True, 0, 0, kind["bf16"],
                                  [out, out2], scale=scale, bias=bias)
torch.cuda.synchronize()
print("done", what)
