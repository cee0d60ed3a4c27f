"""Launch one hot kernel of the data plane a few times at its config size, for
ncu (`-k regex:<kernel> -s <skip> -c 1`):

    python tools/profile_r2.py <what> [batches]

what: f32 | bf16 | u8            C2 collate (B=256 224x224x3) through produce_range
      f32crc | bf16crc | u8crc   the same with the per-batch CRC fused (collate_crc_kernel)
      passthrough                C1 gather (B=64 224x224x3 u8) through produce_range
      llm | llm_persistent       C5 LLM (2048,) int32 B=256 synthetic, per-batch / persistent
                                 (llm_persistent under ncu --set full: the replayed cooperative
                                 launch did not finish in 20 min; use TSB_PT_TRACE instead)
      video                      C5 video (16,3,112,112) u8 B=16 synthetic
      rebatch                    C4 window b=384 straddling two B=512 bf16 slots
      fanout                     one 77 MB slot copied to 2 destinations (same GPU)
      twostage                   stage-1 row gather into 2 input rings + stage-2 restage collate
      crc                        tile CRC-32 of a 154 MB f32 batch
      ingest                     C2 f32 from a PINNED host store: the PCIe gather
                                 (ingest_gather_kernel) + collate, per batch
"""
import sys
import threading

import torch

sys.path.insert(0, ".")
from paper_2409_18749_b200 import (AugmentSpec, CollateLoader, DatasetSpec,  # noqa: E402
                                   StoreSource, SyntheticSource)
from paper_2409_18749_b200 import dataplane as dp  # noqa: E402
from paper_2409_18749_b200._lib import GATE_HOST, ProduceArgs  # noqa: E402
from paper_2409_18749_b200.ring import (DeviceRing, produce_group, produce_range,  # noqa: E402
                                        restage_collate)
from paper_2409_18749_b200.wire import DType  # noqa: E402

what = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 6
torch.cuda.set_device(0)
H, W, C = 224, 224, 3


def run_range(ld, persistent=False, slots=8, crc=False):
    ring = DeviceRing(slots, ld.batch_nbytes, 1, control="host")
    d_crc = torch.zeros(slots, dtype=torch.int32, device="cuda") if crc else None
    a = ld.produce_args(0, with_crc=d_crc)
    a.gate = GATE_HOST
    a.persistent = int(persistent)
    s = torch.cuda.Stream()
    produce_range(ring, a, 1, 0, n, [], stream=s)
    s.synchronize()
    ring.close()


if what.rstrip("crc") in ("f32", "bf16", "u8"):
    dt = {"f32": "float32", "bf16": "bfloat16", "u8": "uint8"}[what.replace("crc", "")]
    store = StoreSource.synthetic(0, 16384, (H, W, C), location="hbm")
    run_range(CollateLoader(DatasetSpec(store, 16384, 256), AugmentSpec(out_dtype=dt)),
              crc=what.endswith("crc"))
elif what == "passthrough":
    store = StoreSource.synthetic(0, 4096, (H, W, C), location="hbm")
    run_range(CollateLoader(DatasetSpec(store, 4096, 64)))
elif what in ("llm", "llm_persistent"):
    ld = CollateLoader(DatasetSpec(SyntheticSource(0, (2048,), DType.I32), 1 << 16, 256))
    run_range(ld, persistent=what == "llm_persistent")
elif what == "video":
    ld = CollateLoader(DatasetSpec(SyntheticSource(0, (16, 3, 112, 112), DType.U8), 4096, 16))
    run_range(ld)
elif what == "rebatch":
    P, b = 512, 384
    store = StoreSource.synthetic(0, 4096, (H, W, C), location="hbm")
    ld = CollateLoader(DatasetSpec(store, 4096, P), AugmentSpec(out_dtype="bfloat16"))
    ring = DeviceRing(3, ld.batch_nbytes, 1, control="host")
    a = ld.produce_args(0)
    a.gate = GATE_HOST
    produce_range(ring, a, 1, 0, 2, [])
    torch.cuda.synchronize()
    in_sb = C * H * W * 2
    out = torch.empty(b * (in_sb + 8), dtype=torch.uint8, device="cuda")
    for _ in range(n):  # window j=1: samples 384..768 = slot 0 [384, 512) + slot 1 [0, 256)
        dp.rebatch_window([ring.slot_ptr(0), ring.slot_ptr(1)], b, b, P, in_sb, 8, out)
    torch.cuda.synchronize()
    ring.close()
elif what == "fanout":
    nbytes = 256 * C * H * W * 2
    src = torch.randint(0, 255, (nbytes,), dtype=torch.uint8, device="cuda")
    dsts = [torch.empty(nbytes, dtype=torch.uint8, device="cuda") for _ in range(2)]
    for _ in range(n):
        dp.fanout(src, dsts, nbytes)
    torch.cuda.synchronize()
elif what == "twostage":
    from paper_2409_18749_b200.collate import _Ingest

    G, B, N = 2, 256, 4096
    store = StoreSource.synthetic(0, N, (H, W, C), location="hbm")
    gld = CollateLoader(DatasetSpec(store, N, B))
    ald = CollateLoader(DatasetSpec(store, N, B), AugmentSpec(out_dtype="float32"))
    in_rings = [DeviceRing(4, gld.batch_nbytes, 1, control="host", writers=G) for _ in range(G)]
    out_rings = [DeviceRing(4, ald.batch_nbytes, 1, control="host") for _ in range(G)]
    tables = [_Ingest(0, B, H * W * C) for _ in range(G)]

    def stage1(g):
        s = torch.cuda.Stream()
        produce_group(in_rings, g, gld.produce_args(0), g, G, 1, 0, n, [[0]] * G, stream=s)
        s.synchronize()

    def stage2(g):
        s = torch.cuda.Stream()
        a = ProduceArgs.from_buffer_copy(ald.produce_args(0))
        a.ingest = tables[g].handle
        a.gate = GATE_HOST
        restage_collate(in_rings[g], 0, out_rings[g], a, 1, n, [0], stream=s)
        s.synchronize()

    def consume(g):
        r = out_rings[g]
        for q in range(1, n + 1):
            r.host_wait_ready(r.slot_of(q), q, timeout_s=60)
            r.host_ack(0, q)

    for r in in_rings + out_rings:
        r.set_cursor(0, 0)
    ts = [threading.Thread(target=f, args=(g,)) for f in (stage1, stage2, consume)
          for g in range(G)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(120)
elif what == "crc":
    nbytes = 256 * C * H * W * 4 + 2048
    data = torch.randint(0, 255, (nbytes,), dtype=torch.uint8, device="cuda")
    out = torch.zeros(1, dtype=torch.int32, device="cuda")
    for _ in range(n):
        dp.crc32(data, nbytes, out)
    torch.cuda.synchronize()
elif what == "ingest":
    store = StoreSource.synthetic(0, 4096, (H, W, C), location="pinned")
    run_range(CollateLoader(DatasetSpec(store, 4096, 256), AugmentSpec(out_dtype="float32")))
else:
    raise SystemExit(f"unknown target {what}")
print("done", what)
