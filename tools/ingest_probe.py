"""Pinned-store ingest throughput on the e2e workload without the facade:
CollateLoader(pinned StoreSource) through the native producer loop (staged
ingest gather kernel + fused collate with the checksum), no consumers, K
batches; H2D GB/s = the bytes the ingest moved / device time.

    TSB_IG_CHUNK=16384 python tools/ingest_probe.py [K]
"""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2409_18749_b200 import AugmentSpec, CollateLoader, DatasetSpec, StoreSource  # noqa: E402
from paper_2409_18749_b200 import dataplane as dp  # noqa: E402
from paper_2409_18749_b200._lib import GATE_HOST  # noqa: E402
from paper_2409_18749_b200.ring import DeviceRing, produce_range  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 96
B, N, SLOTS = 256, 16384, 8
torch.cuda.set_device(0)
store = StoreSource.synthetic(0, N, (224, 224, 3), location="pinned")
ld = CollateLoader(DatasetSpec(store, N, B), AugmentSpec(out_dtype="float32"))
ring = DeviceRing(SLOTS, ld.batch_nbytes, 1, control="host")
d_crc = torch.zeros(SLOTS, dtype=torch.int32, device="cuda")
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
        produce_range(ring, a, q, bi, m, [], stream=s)
        done += m


run(1, 8)
s.synchronize()
b0 = ld._ingest.bytes_enqueued()
e0, e1 = dp.DeviceEvent(), dp.DeviceEvent()
e0.record(s)
run(9, K)
e1.record(s)
s.synchronize()
ms = e0.elapsed_ms(e1)
moved = ld._ingest.bytes_enqueued() - b0
print(json.dumps({"chunk": int(os.environ.get("TSB_IG_CHUNK", "16384")), "batches": K,
                  "ms_per_batch": round(ms / K, 3), "h2d_gbs": round(moved / (ms / 1e3) / 1e9, 1),
                  "produced_samples_s": round(B * K / (ms / 1e3), 1)}))
ring.close()
