"""Launch the fused passthrough producer (C1 shape) a few times through
produce_range, for ncu: python tools/profile_passthrough.py [batches]."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2409_18749_b200 import CollateLoader, DatasetSpec, StoreSource  # noqa: E402
from paper_2409_18749_b200._lib import GATE_HOST  # noqa: E402
from paper_2409_18749_b200.ring import DeviceRing, produce_range  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 6
torch.cuda.set_device(0)
store = StoreSource.synthetic(0, 4096, (224, 224, 3))
ld = CollateLoader(DatasetSpec(store, 4096, 64))
ring = DeviceRing(8, ld.batch_nbytes, 1, control="host")
a = ld.produce_args(0)
a.gate = GATE_HOST
s = torch.cuda.Stream()
produce_range(ring, a, 1, 0, n, [], stream=s)
s.synchronize()
ring.close()
print("done")
