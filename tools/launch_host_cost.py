"""Host time of one tsb_produce_range(n=1) call (gate open, device far behind
the host): the fused collate+CRC launch vs the plain collate launch.

    python tools/launch_host_cost.py [calls]"""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2409_18749_b200 import AugmentSpec, CollateLoader, DatasetSpec, StoreSource  # noqa: E402
from paper_2409_18749_b200._lib import GATE_HOST  # noqa: E402
from paper_2409_18749_b200.ring import DeviceRing, produce_range  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 48
torch.cuda.set_device(0)
store = StoreSource.synthetic(0, 16384, (224, 224, 3), location="hbm")
ld = CollateLoader(DatasetSpec(store, 16384, 256), AugmentSpec(out_dtype="float32"))
ring = DeviceRing(K + 8, ld.batch_nbytes, 1, control="host")
for crc in (True, False, True, False):
    d_crc = torch.zeros(K + 8, dtype=torch.int32, device="cuda") if crc else None
    s = torch.cuda.Stream()
    a = ld.produce_args(0, with_crc=d_crc)
    a.gate = GATE_HOST
    produce_range(ring, a, 1, 0, 1, [], stream=s)
    s.synchronize()
    ts = []
    for q in range(2, K + 2):
        a.chain = 1
        t0 = time.perf_counter()
        produce_range(ring, a, q, (q - 1) % len(ld), 1, [], stream=s)
        ts.append((time.perf_counter() - t0) * 1e6)
    s.synchronize()
    ts.sort()
    print(json.dumps({"checksum": crc, "median_host_us": round(ts[len(ts) // 2], 2),
                      "min_host_us": round(ts[0], 2)}), flush=True)
ring.close()
