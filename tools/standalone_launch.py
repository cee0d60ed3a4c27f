"""Device time of ONE produce_range(n=1) launch when the stream is idle before
it (no PDL overlap with a previous batch) -- the facade's situation when its
host loop is slower than the device.  C2 f32 / bf16, checksum on and off.

    python tools/standalone_launch.py [reps]"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2409_18749_b200 import AugmentSpec, CollateLoader, DatasetSpec, StoreSource  # noqa: E402
from paper_2409_18749_b200 import dataplane as dp  # noqa: E402
from paper_2409_18749_b200._lib import GATE_HOST  # noqa: E402
from paper_2409_18749_b200.ring import DeviceRing, produce_range  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 64
torch.cuda.set_device(0)
store = StoreSource.synthetic(0, 16384, (224, 224, 3), location="hbm")
for kind in ("float32", "bfloat16"):
    ld = CollateLoader(DatasetSpec(store, 16384, 256), AugmentSpec(out_dtype=kind))
    ring = DeviceRing(8, ld.batch_nbytes, 1, control="host")
    for crc in (True, False):
        d_crc = torch.zeros(8, dtype=torch.int32, device="cuda") if crc else None
        s = torch.cuda.Stream()
        ts = []
        for q in range(1, R + 1):
            a = ld.produce_args(0, with_crc=d_crc)
            a.gate = GATE_HOST
            e0, e1 = dp.DeviceEvent(), dp.DeviceEvent()
            e0.record(s)
            produce_range(ring, a, q, (q - 1) % len(ld), 1, [], stream=s)
            e1.record(s)
            s.synchronize()
            if q > 4:
                ts.append(e0.elapsed_ms(e1) * 1e3)
        ts.sort()
        print(json.dumps({"kind": kind, "checksum": crc, "median_us": round(ts[len(ts) // 2], 2),
                          "min_us": round(ts[0], 2)}), flush=True)
    ring.close()
