"""Diagnostics for the persistent range kernel: every batch's parity status
(fraction of bytes right / zero, CRC vs zlib) instead of stopping at the first
mismatch.  python tools/ccrange_diag.py [dtype c B n slots h w]"""
import sys
import threading
import zlib

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle  # noqa: E402
from paper_2409_18749_b200 import AugmentSpec, CollateLoader, DatasetSpec, StoreSource  # noqa: E402
from paper_2409_18749_b200._lib import GATE_HOST  # noqa: E402
from paper_2409_18749_b200.ring import DeviceRing, produce_range  # noqa: E402

a = sys.argv[1:]
dt = a[0] if a else "uint8"
c, B, n, S = (int(x) for x in (a[1:5] if len(a) > 4 else (1, 33, 7, 4)))
h, w = (int(x) for x in (a[5:7] if len(a) > 6 else (64, 64)))
persist = int(a[7]) if len(a) > 7 else 1
N, pad, seed, aug_seed = 60, 6, 3, 5
KIND = {"float32": 1, "bfloat16": 2, "uint8": 0}[dt]
store = StoreSource.synthetic(seed, N, (h, w, c))
ld = CollateLoader(DatasetSpec(store, N, B, shuffle_seed=2),
                   AugmentSpec(pad=pad, flip=True, out_dtype=dt, seed=aug_seed))
ring = DeviceRing(S, ld.batch_nbytes, 1, control="host")
ring.set_cursor(0, 0)
d_crc = torch.zeros(S, dtype=torch.int32, device="cuda")
got = {}


def consumer():
    cs = torch.cuda.Stream()
    for q in range(1, n + 1):
        slot = ring.slot_of(q)
        ring.host_wait_ready(slot, q, timeout_s=300)
        with torch.cuda.stream(cs):
            raw = ring.view(slot, (ld.batch_nbytes,), torch.uint8).cpu().numpy().copy()
            crc = int(d_crc[slot].item()) & 0xFFFFFFFF
        got[q] = (raw, crc)
        ring.host_ack(0, q)


t = threading.Thread(target=consumer)
t.start()
ps = torch.cuda.Stream()
L = len(ld)
q = 1
while q <= n:
    epoch, bi = divmod(q - 1, L)
    m = min(n - q + 1, L - bi)
    pa = ld.produce_args(epoch, with_crc=d_crc)
    pa.gate = GATE_HOST
    pa.persistent = persist
    produce_range(ring, pa, q, bi, m, [0], stream=ps)
    q += m
ps.synchronize()
t.join(300)
store_h = oracle.make_store(seed, N, h * w * c)
scale, bias = oracle.norm_consts()
for q in range(1, n + 1):
    raw, crc = got[q]
    epoch, bi = divmod(q - 1, L)
    idx = oracle.epoch_order(N, 2, epoch)[bi * B:(bi + 1) * B]
    want = oracle.collate_augment(store_h, idx, h, w, c, pad, True, aug_seed, epoch, KIND,
                                  scale if KIND else None, bias if KIND else None)
    x = raw[:ld.input_nbytes]
    wb = np.frombuffer(want.tobytes(), np.uint8)
    eq = float((x == wb).mean())
    zero = float((x == 0).mean())
    body = raw[:ld.input_nbytes + 8 * B].tobytes()
    tgt_ok = np.array_equal(np.frombuffer(raw[ld.input_nbytes:ld.input_nbytes + 8 * B].tobytes(), "<i8"), idx)
    bad = np.nonzero(x != wb)[0]
    print(f"q={q} slot={ring.slot_of(q)} eq={eq:.4f} zero={zero:.4f} tgt_ok={tgt_ok} "
          f"crc_ok={crc == zlib.crc32(body)} first_bad={bad[:1].tolist()} last_bad={bad[-1:].tolist()}",
          flush=True)
ring.close()
