"""Per-batch device time of the C2/C3 collate through the native producer loop,
with the per-batch CRC-32 (fused into the collate kernel when the geometry
allows) and without -- B=256 224x224x3 from an HBM store, no consumers,
PDL-chained launches, CUDA events on the producer stream.

    python tools/crc_fused_timing.py [kinds] [batches]     (kinds: f32,bf16,u8)

Prints one JSON line per (kind, checksum).  Env knobs of the kernels apply
(TSB_CC_DEBUG, TSB_CRC_FUSED, ...)."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2409_18749_b200 import AugmentSpec, CollateLoader, DatasetSpec, StoreSource  # noqa: E402
from paper_2409_18749_b200 import dataplane as dp  # noqa: E402
from paper_2409_18749_b200._lib import GATE_HOST  # noqa: E402
from paper_2409_18749_b200.ring import DeviceRing, produce_range  # noqa: E402

kinds = (sys.argv[1] if len(sys.argv) > 1 else "f32,bf16,u8").split(",")
K = int(sys.argv[2]) if len(sys.argv) > 2 else 256
H = W = 224
C, N, SLOTS = 3, 16384, 8
B = int(os.environ.get("TIMING_B", "256"))
PERSIST = int(os.environ.get("TIMING_PERSIST", "0"))  # 1: one persistent launch per range
torch.cuda.set_device(0)
store = StoreSource.synthetic(0, N, (H, W, C), location="hbm")
E = {"f32": 4, "bf16": 2, "u8": 1}
for kind in kinds:
    dt = {"f32": "float32", "bf16": "bfloat16", "u8": "uint8"}[kind]
    ld = CollateLoader(DatasetSpec(store, N, B), AugmentSpec(out_dtype=dt))
    ring = DeviceRing(SLOTS, ld.batch_nbytes, 1, control="host")
    for crc in (True, False):
        d_crc = torch.zeros(SLOTS, dtype=torch.int32, device="cuda") if crc else None
        s = torch.cuda.Stream()
        L = len(ld)

        def run(q0, n):
            done = 0
            while done < n:
                q = q0 + done
                epoch, bi = divmod(q - 1, L)
                m = min(n - done, L - bi)
                a = ld.produce_args(epoch, with_crc=d_crc)
                a.gate = GATE_HOST
                a.persistent = PERSIST if crc else 0
                produce_range(ring, a, q, bi, m, [], stream=s)
                if os.environ.get("TIMING_SYNC"):
                    print("range", q, bi, m, flush=True)
                    s.synchronize()
                    print("  done", flush=True)
                done += m

        run(1, 8)
        s.synchronize()
        e0, e1 = dp.DeviceEvent(), dp.DeviceEvent()
        e0.record(s)
        run(9, K)
        e1.record(s)
        s.synchronize()
        ms = e0.elapsed_ms(e1) / K
        alg = B * (H * W * C + C * H * W * E[kind])
        print(json.dumps({"kind": kind, "b": B, "checksum": crc, "persistent": PERSIST, "us_per_batch": round(ms * 1e3, 2),
                          "alg_gbs": round(alg / (ms / 1e3) / 1e9, 1)}),
              flush=True)
    ring.close()
