"""Batch CRC-32 fused into the collate kernel (tsb_collate_crc.cuh).

The reference checksums every segment it creates (bs/payload.py:218,
``crc32(mv)`` over the whole payload) and the Announce carries it.  Here the
collate kernel's checksum warps compute it from the staged source bytes and
the completing CTA writes the zlib CRC-32 of the slot (input + int64 target)
into ``d_crc[slot]``.  Every case checks that word against ``zlib.crc32`` of
the slot bytes AND the slot bytes against the oracle's collate, across the
output kinds, channel counts, crop pads (rows and columns cropped out
entirely), flips, batch sizes that leave the target lanes ragged, a full C2
batch, and geometries the fused kernel does not take (separate CRC kernel)."""

import threading
import time
import zlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2409_18749_b200 import AugmentSpec, CollateLoader, DatasetSpec, StoreSource  # noqa: E402
from paper_2409_18749_b200._lib import GATE_HOST  # noqa: E402
from paper_2409_18749_b200.ring import DeviceRing, produce_range  # noqa: E402

KIND = {"float32": 1, "bfloat16": 2, "uint8": 0}


def _run(oracle, h, w, c, B, N, pad, out_dtype, n, with_target=True, seed=3, aug_seed=5,
         crc_at_ready=True, slots=3, persistent=False, consumer_delay=0.0):
    """n batches through the native producer loop with a per-batch CRC.  The
    fused kernel's CRC is in d_crc[slot] when the slot is published, and the
    consumer reads it then (crc_at_ready); the separate CRC kernel runs after
    the publish, so those cases keep n <= slots and read it at the end."""
    store = StoreSource.synthetic(seed, N, (h, w, c))
    ld = CollateLoader(DatasetSpec(store, N, B, shuffle_seed=2),
                       AugmentSpec(pad=pad, flip=True, out_dtype=out_dtype, seed=aug_seed),
                       with_target=with_target)
    S = slots if crc_at_ready else n
    ring = DeviceRing(S, ld.batch_nbytes, 1, control="host")
    ring.set_cursor(0, 0)
    d_crc = torch.zeros(S, dtype=torch.int32, device="cuda")
    got = {}
    errs = []

    def consumer():
        try:
            cs = torch.cuda.Stream()
            for q in range(1, n + 1):
                slot = ring.slot_of(q)
                ring.host_wait_ready(slot, q, timeout_s=120)
                if consumer_delay:
                    time.sleep(consumer_delay)
                with torch.cuda.stream(cs):
                    raw = ring.view(slot, (ld.batch_nbytes,), torch.uint8).cpu().numpy().copy()
                    crc = int(d_crc[slot].item()) & 0xFFFFFFFF if crc_at_ready else None
                got[q] = (raw, crc)
                ring.host_ack(0, q)
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    t = threading.Thread(target=consumer)
    t.start()
    ps = torch.cuda.Stream()
    L = len(ld)
    q = 1
    while q <= n:
        epoch, bi = divmod(q - 1, L)
        m = min(n - q + 1, L - bi)
        a = ld.produce_args(epoch, with_crc=d_crc)
        a.gate = GATE_HOST
        a.persistent = int(persistent)
        produce_range(ring, a, q, bi, m, [0], stream=ps)
        q += m
    ps.synchronize()
    t.join(120)
    assert not t.is_alive() and not errs, errs
    store_h = oracle.make_store(seed, N, h * w * c)
    scale, bias = oracle.norm_consts()
    kind = KIND[out_dtype]
    for q in range(1, n + 1):
        raw, crc = got[q]
        if not crc_at_ready:
            crc = int(d_crc[ring.slot_of(q)].item()) & 0xFFFFFFFF
        epoch, bi = divmod(q - 1, L)
        idx = oracle.epoch_order(N, 2, epoch)[bi * B:(bi + 1) * B]
        want = oracle.collate_augment(store_h, idx, h, w, c, pad, True, aug_seed, epoch, kind,
                                      scale if kind else None, bias if kind else None)
        assert raw[:ld.input_nbytes].tobytes() == want.tobytes(), q
        body = raw[:ld.input_nbytes + (8 * B if with_target else 0)].tobytes()
        assert crc == zlib.crc32(body), (q, hex(crc), hex(zlib.crc32(body)))
    ring.close()
    return ld


@pytest.mark.parametrize("out_dtype", ["float32", "bfloat16", "uint8"])
@pytest.mark.parametrize("c", [3, 1])
def test_fused_crc_matches_zlib(oracle, out_dtype, c):
    _run(oracle, 64, 96, c, 8, 40, 6, out_dtype, 7)


@pytest.mark.parametrize("B", [1, 31, 33, 37])
def test_fused_crc_ragged_target_lanes(oracle, B):
    """b not a multiple of 32: the target's lanes start on virtual zeros."""
    _run(oracle, 32, 64, 3, B, 80, 4, "float32", 3)


@pytest.mark.parametrize("pad", [0, 40])
def test_fused_crc_crop_extremes(oracle, pad):
    """pad 0 (no crop) and pad > h (samples cropped out entirely: zero rows)."""
    _run(oracle, 32, 32, 3, 5, 20, pad, "bfloat16", 5)


def test_fused_crc_without_target(oracle):
    _run(oracle, 64, 64, 3, 6, 24, 8, "float32", 4, with_target=False)


@pytest.mark.parametrize("h,w", [(40, 40), (33, 64), (48, 36)])
def test_unfused_geometries_still_checksummed(oracle, h, w):
    """w % 32 != 0 or h not a whole number of row blocks: the collate runs
    alone and the separate CRC kernel follows -- same CRC."""
    _run(oracle, h, w, 3, 4, 16, 5, "float32", 4, crc_at_ready=False)


def test_fused_crc_full_c2_batch(oracle):
    """C2 at size: B=256 224x224x3 -> f32 NCHW (154 MB + 2 KB target)."""
    _run(oracle, 224, 224, 3, 256, 1024, 16, "float32", 2)


def test_fused_kernel_is_the_one_that_runs():
    """The profiler sees collate_crc_kernel (not collate + crc_tile) when a
    checksum is requested for a fusable geometry."""
    from torch.profiler import ProfilerActivity, profile

    h = w = 64
    B, N = 8, 32
    ld = CollateLoader(DatasetSpec(StoreSource.synthetic(1, N, (h, w, 3)), N, B),
                       AugmentSpec(pad=4, flip=True, out_dtype="float32"))
    ring = DeviceRing(2, ld.batch_nbytes, 1, control="host")
    d_crc = torch.zeros(2, dtype=torch.int32, device="cuda")
    a = ld.produce_args(0, with_crc=d_crc)
    a.gate = GATE_HOST
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        produce_range(ring, a, 1, 0, 1, [])
        torch.cuda.synchronize()
    names = [e.name for e in prof.events() if e.device_type.name == "CUDA"]
    assert any("collate_crc_kernel" in n for n in names), names
    assert not any("crc_tile_kernel" in n or "crc_kernel" == n for n in names), names
    ring.close()


@pytest.mark.parametrize("out_dtype,c,B,n,slots", [
    ("float32", 3, 8, 9, 3), ("bfloat16", 3, 5, 12, 2), ("uint8", 1, 33, 7, 4),
    ("float32", 3, 1, 16, 3),
])
def test_persistent_range_crc(oracle, out_dtype, c, B, n, slots):
    """One cooperative launch for the range (collate_crc_range_kernel): the
    slot gate runs on the device against the consumer's acks, batches cross
    CTA boundaries mid-stage, every slot's CRC is in place at its publish.
    B=1: a batch of 2 items (fewer items than CTAs)."""
    _run(oracle, 64, 64, c, B, 60, 6, out_dtype, n, slots=slots, persistent=True)


def test_persistent_range_crc_full_c2(oracle):
    """C2 geometry, 6 batches through a 2-slot ring in one launch."""
    _run(oracle, 224, 224, 3, 256, 1024, 16, "float32", 6, slots=2, persistent=True)


def test_persistent_range_crc_epoch_boundary(oracle):
    """A range that crosses the epoch (the loop splits it: one launch per epoch chunk)."""
    _run(oracle, 32, 64, 3, 4, 12, 4, "float32", 7, persistent=True)


@pytest.mark.parametrize("persistent", [False, True])
def test_epoch_orders_outlive_queued_launches(oracle, persistent):
    """One batch per epoch and a slow consumer: the producer enqueues launches
    for later epochs while earlier ones still wait on the slot gate, and each
    epoch switch drops the previous epoch's device order.  The order buffers
    must stay allocated for the queued launches (ring.hold_for_stream), or the
    next epoch's order lands in the same block and they gather wrong samples."""
    _run(oracle, 32, 64, 3, 33, 60, 4, "float32", 10, slots=2, persistent=persistent,
         consumer_delay=0.05)
