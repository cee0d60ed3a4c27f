"""Native producer/consumer loops (tsb_produce_range / tsb_consume_range) over
the device ring, incl. the collate kernel's fused epilogue (target copy +
slot publish from the last CTA) and the host-shared control block."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2409_18749_b200 import (AugmentSpec, CollateLoader, DatasetSpec,  # noqa: E402
                                   StoreSource, SyntheticSource)
from paper_2409_18749_b200.ring import DeviceRing, consume_range, produce_range  # noqa: E402
from paper_2409_18749_b200.wire import DType  # noqa: E402


def _snapshots(ld, ring, n, epoch=0, stride=1):
    """Produce n batches through the native loop; one in-process consumer
    stream snapshots each slot between wait_ready and ack."""
    ps, cs = torch.cuda.Stream(), torch.cuda.Stream()
    ring.set_cursor(0, epoch * len(ld))  # admitted at the epoch start (producer.py semantics)
    args = ld.produce_args(epoch)
    args.wait_stride = stride
    produce_range(ring, args, epoch * len(ld) + 1, 0, n, [0], stream=ps)
    snaps = []
    for i in range(n):
        q = epoch * len(ld) + 1 + i
        slot = ring.slot_of(q)
        with torch.cuda.stream(cs):
            ring.wait_ready(slot, q, cs)
            snaps.append(ring.view(slot, (ld.batch_nbytes,), torch.uint8).clone())
            ring.ack(0, q, cs)
    torch.cuda.synchronize()
    return [s.cpu().numpy() for s in snaps]


@pytest.mark.parametrize("control,stride", [("device", 1), ("host", 1), ("host", 2)])
@pytest.mark.parametrize("out_dtype,kind", [("float32", 1), ("bfloat16", 2), ("uint8", 0)])
def test_produce_range_augment_fused_publish(oracle, control, stride, out_dtype, kind):
    h, w, c, B, N = 32, 64, 3, 8, 96
    store = StoreSource.synthetic(3, N, (h, w, c))
    ld = CollateLoader(DatasetSpec(store, N, B, shuffle_seed=5),
                       AugmentSpec(pad=4, flip=True, out_dtype=out_dtype, seed=9))
    ring = DeviceRing(3, ld.batch_nbytes, 1, control=control)
    snaps = _snapshots(ld, ring, 10, epoch=1, stride=stride)
    store_h = oracle.make_store(3, N, h * w * c)
    order = oracle.epoch_order(N, 5, 1)
    scale, bias = oracle.norm_consts()
    for i, snap in enumerate(snaps):
        idx = order[i * B:(i + 1) * B]
        want = oracle.collate_augment(store_h, idx, h, w, c, 4, True, 9, 1, kind,
                                      scale if kind else None, bias if kind else None)
        assert snap[:ld.input_nbytes].tobytes() == want.tobytes()
        np.testing.assert_array_equal(snap[ld.input_nbytes:].view(np.int64), idx)
    assert ring.read_ready(ring.slot_of(len(ld) + 10)) == len(ld) + 10
    ring.close()


@pytest.mark.parametrize("mode", ["gather", "synthetic"])
def test_produce_range_passthrough(golden, mode):
    case = golden["prepare_batch"][0]  # 224x224x3 u8 B=64 N=1024 epoch 0
    if mode == "synthetic":
        src = SyntheticSource(0, (224, 224, 3), DType.U8)
    else:  # epoch 0 store == synthetic epoch 0 (DirectorySource semantics)
        src = StoreSource.synthetic(0, 1024, (224, 224, 3))
    ld = CollateLoader(DatasetSpec(src, 1024, 64, shuffle_seed=0))
    ring = DeviceRing(2, ld.batch_nbytes, 1, control="host")
    snaps = _snapshots(ld, ring, 4)
    import zlib

    assert zlib.crc32(snaps[0][:ld.input_nbytes].tobytes()) == case["crc32"]
    assert zlib.crc32(snaps[3][:ld.input_nbytes].tobytes()) == golden["prepare_batch"][1]["crc32"]
    np.testing.assert_array_equal(snaps[0][ld.input_nbytes:].view(np.int64), case["indices"])
    ring.close()


def test_host_consumer_ops_and_eviction():
    ring = DeviceRing(2, 1 << 16, 2, control="host")
    s = torch.cuda.Stream()
    ring.publish(1, 7, s)
    s.synchronize()
    ring.host_wait_ready(1, 7, timeout_s=5)
    with pytest.raises(Exception):
        ring.host_wait_ready(0, 1, timeout_s=0.01)
    ring.host_ack(0, 5)
    assert ring.read_cursor(0) == 5
    # a device wait on an evicted consumer must not wedge the stream
    ring.wait_free([0, 1], 9, s)
    ring.evict(1)
    ring.host_ack(0, 9)
    s.synchronize()
    ring.close()


def test_consume_range_events():
    from paper_2409_18749_b200 import dataplane as dp

    ring = DeviceRing(4, 4096, 1)
    ps, cs = torch.cuda.Stream(), torch.cuda.Stream()
    e0, e1 = dp.DeviceEvent(), dp.DeviceEvent()
    consume_range(ring, 0, 1, 8, events=[e0, e1], stream=cs)
    for q in range(1, 9):
        ring.wait_free([0], q - 4, ps)
        ring.publish(ring.slot_of(q), q, ps)
    cs.synchronize()
    assert ring.read_cursor(0) == 8 and e0.elapsed_ms(e1) >= 0
    ring.close()


@pytest.mark.parametrize("out_dtype,kind", [("float32", 1), ("bfloat16", 2)])
def test_host_gate_pdl_chain_with_concurrent_consumer(oracle, out_dtype, kind):
    """TSB_GATE_HOST: the producer thread blocks on the host-shared cursors and
    the stream carries only PDL-chained fused kernels.  A host consumer thread
    (map-and-ack, bs/cli.py:252-258) checks every batch against the oracle
    before releasing it -- a slot overwritten early would show up as a mismatch
    -- and its ack is what lets the producer run ahead."""
    import threading

    from paper_2409_18749_b200._lib import GATE_HOST

    h, w, c, B, N, S, n = 32, 64, 3, 8, 96, 3, 24
    store = StoreSource.synthetic(4, N, (h, w, c))
    ld = CollateLoader(DatasetSpec(store, N, B, shuffle_seed=2),
                       AugmentSpec(pad=4, flip=True, out_dtype=out_dtype, seed=1))
    ring = DeviceRing(S, ld.batch_nbytes, 2, control="host")
    ring.set_cursor(0, 0)
    ring.evict(1)  # a dead consumer slot must not block the host gate
    store_h = oracle.make_store(4, N, h * w * c)
    scale, bias = oracle.norm_consts()
    L = len(ld)
    errors = []

    def consumer():
        try:
            for q in range(1, n + 1):
                epoch, bi = divmod(q - 1, L)
                slot = ring.slot_of(q)
                ring.host_wait_ready(slot, q, timeout_s=60)
                got = ring.view(slot, (ld.batch_nbytes,), torch.uint8).cpu().numpy()
                idx = oracle.epoch_order(N, 2, epoch)[bi * B:(bi + 1) * B]
                want = oracle.collate_augment(store_h, idx, h, w, c, 4, True, 1, epoch, kind,
                                              scale, bias)
                if got[:ld.input_nbytes].tobytes() != want.tobytes():
                    errors.append(q)
                ring.host_ack(0, q)
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e))
            ring.evict(0)

    t = threading.Thread(target=consumer)
    t.start()
    ps = torch.cuda.Stream()
    q = 1
    while q <= n:
        epoch, bi = divmod(q - 1, L)
        m = min(n - q + 1, L - bi)
        a = ld.produce_args(epoch)
        a.gate = GATE_HOST
        produce_range(ring, a, q, bi, m, [0, 1], stream=ps)
        q += m
    ps.synchronize()
    t.join(120)
    assert not t.is_alive() and not errors, errors
    assert ring.read_cursor(0) == n
    ring.close()


def test_host_gate_needs_host_control():
    from paper_2409_18749_b200._lib import GATE_HOST

    store = StoreSource.synthetic(0, 16, (8, 16, 3))
    ld = CollateLoader(DatasetSpec(store, 16, 4), AugmentSpec(pad=2, out_dtype="float32"))
    ring = DeviceRing(2, ld.batch_nbytes, 1, control="device")
    a = ld.produce_args(0)
    a.gate = GATE_HOST
    with pytest.raises(ValueError, match="host control"):
        produce_range(ring, a, 1, 0, 1, [0])
    ring.close()


@pytest.mark.parametrize("mode,h,pad", [("augment_f32", 32, 4), ("augment_bf16", 32, 4),
                                        ("gather", 32, 4), ("augment_f32", 8, 12),
                                        ("augment_u8", 24, 24)])
def test_staged_copy_engine_ingest_from_pinned_store(oracle, mode, h, pad):
    """Pinned-host store: each batch's scattered sample rows cross PCIe by the
    one gather kernel over the mapped pinned store) into HBM staging (augment) or straight
    into the slot (gather); results identical to the oracle.  Augment
    batches copy only the rows the crop reads (the staging buffers keep the
    previous batches' other rows, which the kernel must never read) -- down
    to samples cropped out entirely when pad >= h."""
    from paper_2409_18749_b200._lib import GATE_HOST

    w, c, B, N, S, n = 64, 3, 8, 64, 3, 12
    store = StoreSource.synthetic(9, N, (h, w, c), location="pinned")
    out_dtype = {"augment_f32": "float32", "augment_bf16": "bfloat16", "augment_u8": "uint8"}
    aug = None if mode == "gather" else AugmentSpec(pad=pad, flip=True, out_dtype=out_dtype[mode],
                                                    seed=2)
    ld = CollateLoader(DatasetSpec(store, N, B, shuffle_seed=1), aug)
    ring = DeviceRing(S, ld.batch_nbytes, 1, control="host")
    ring.set_cursor(0, 0)
    store_h = oracle.make_store(9, N, h * w * c)
    scale, bias = oracle.norm_consts()
    kind = {"augment_f32": 1, "augment_bf16": 2, "augment_u8": 0}.get(mode)
    L = len(ld)
    got = {}
    import threading

    def consumer():
        for q in range(1, n + 1):
            slot = ring.slot_of(q)
            ring.host_wait_ready(slot, q, timeout_s=60)
            got[q] = ring.view(slot, (ld.batch_nbytes,), torch.uint8).cpu().numpy().copy()
            ring.host_ack(0, q)

    t = threading.Thread(target=consumer)
    t.start()
    ps = torch.cuda.Stream()
    q = 1
    while q <= n:
        epoch, bi = divmod(q - 1, L)
        m = min(n - q + 1, L - bi)
        a = ld.produce_args(epoch)
        assert a.ingest and a.h_order
        a.gate = GATE_HOST
        produce_range(ring, a, q, bi, m, [0], stream=ps)
        q += m
    ps.synchronize()
    t.join(60)
    assert not t.is_alive()
    for q in range(1, n + 1):
        epoch, bi = divmod(q - 1, L)
        idx = oracle.epoch_order(N, 1, epoch)[bi * B:(bi + 1) * B]
        if kind is None:
            want = oracle.gather(store_h, idx, h * w * c)
        else:
            want = oracle.collate_augment(store_h, idx, h, w, c, pad, True, 2, epoch, kind,
                                          scale, bias)
        assert got[q][:ld.input_nbytes].tobytes() == want.tobytes(), q
        np.testing.assert_array_equal(got[q][ld.input_nbytes:].view(np.int64), idx)
    sent = ld._ingest.bytes_enqueued() - 8 * B * n  # less the index uploads
    if kind is None:
        assert sent == n * B * h * w * c
    else:  # the rows the crop reads widened to whole 128-byte lines, plus the param rows
        rows, line, sb, rb = 0, 128, h * w * c, w * c
        for q in range(1, n + 1):
            epoch, bi = divmod(q - 1, L)
            idx = oracle.epoch_order(N, 1, epoch)[bi * B:(bi + 1) * B]
            for oy in oracle.aug_params(2, epoch, idx, pad)[:, 0].astype(np.int64):
                lo, hi = max(oy - pad, 0), min(h + oy - pad, h)
                if hi > lo:  # cropped-out sample: no bytes
                    b0 = (lo * rb) // line * line
                    b1 = min(-(-(hi * rb) // line) * line, sb)
                    rows += b1 - b0
        assert sent == rows + 12 * B * n
    ring.close()


@pytest.mark.parametrize("mode", ["gather", "synthetic"])
def test_persistent_producer_matches_reference(golden, mode):
    """One cooperative persistent launch produces a whole range of batches,
    gating each slot on the host-shared cursors from the device; a host
    consumer (map-and-ack) checks every batch against the reference's CRCs."""
    import threading
    import zlib

    from paper_2409_18749_b200._lib import GATE_HOST

    cases = {(c["epoch"], c["batch_index"]): c for c in golden["prepare_batch"]
             if c["name"] == "img_b64"}
    if mode == "synthetic":
        src = SyntheticSource(0, (224, 224, 3), DType.U8)
    else:
        src = StoreSource.synthetic(0, 1024, (224, 224, 3))
    ld = CollateLoader(DatasetSpec(src, 1024, 64, shuffle_seed=0))
    ring = DeviceRing(3, ld.batch_nbytes, 2, control="host")  # 3 slots: forces device-side gating
    ring.set_cursor(0, 0)
    ring.evict(1)
    L, n = len(ld), 16
    crcs = {}

    def consumer():
        for q in range(1, n + 1):
            s = ring.slot_of(q)
            ring.host_wait_ready(s, q, timeout_s=60)
            v = ring.view(s, (ld.batch_nbytes,), torch.uint8).cpu().numpy()
            crcs[q] = (zlib.crc32(v[:ld.input_nbytes].tobytes()),
                       v[ld.input_nbytes:].view(np.int64).copy())
            ring.host_ack(0, q)

    t = threading.Thread(target=consumer)
    t.start()
    a = ld.produce_args(0)
    a.gate = GATE_HOST
    a.persistent = 1
    ps = torch.cuda.Stream()
    produce_range(ring, a, 1, 0, n, [0, 1], stream=ps)
    ps.synchronize()
    t.join(60)
    assert not t.is_alive() and len(crcs) == n
    assert L >= n
    for (e, bi), c in cases.items():
        if e == 0 and bi < n:
            assert crcs[bi + 1][0] == c["crc32"]
    np.testing.assert_array_equal(crcs[1][1], cases[(0, 0)]["indices"])
    a.persistent = 0
    ring.close()


def test_ring_operations_leave_the_current_device_alone():
    """Entry points that work on a ring's device (creation, host-control
    attach, stream memops) give the caller's current device back (on a
    one-GPU box this checks the plumbing; the guard matters with several)."""
    torch.cuda.set_device(0)
    before = torch.cuda.current_device()
    ring = DeviceRing(2, 4096, 1, device=0, control="host")
    s = torch.cuda.Stream()
    ring.publish(0, 1, s)
    ring.ack(0, 1, s)
    s.synchronize()
    assert torch.cuda.current_device() == before
    ring.close()


def test_persistent_producer_pipelines_small_batches(oracle):
    """C5 LLM shape through the persistent producer: many small batches whose
    work items run concurrently across slots (no grid-wide batch boundary);
    with only 4 slots every reuse is gated on the host consumer's release.
    Each batch is checked (CRC of the slot before releasing it) against the
    oracle's synthetic fill of the same indices (bs/pipeline.py:183-189)."""
    import threading
    import zlib

    from paper_2409_18749_b200._lib import GATE_HOST

    N, B, n = 1 << 14, 256, 48
    ld = CollateLoader(DatasetSpec(SyntheticSource(3, (2048,), DType.I32), N, B, shuffle_seed=4))
    ring = DeviceRing(4, ld.batch_nbytes, 1, control="host")
    ring.set_cursor(0, 0)
    got = {}

    def consumer():
        for q in range(1, n + 1):
            s = ring.slot_of(q)
            ring.host_wait_ready(s, q, timeout_s=60)
            v = ring.view(s, (ld.batch_nbytes,), torch.uint8).cpu().numpy()
            got[q] = (zlib.crc32(v[:ld.input_nbytes].tobytes()),
                      v[ld.input_nbytes:].view(np.int64).copy())
            ring.host_ack(0, q)

    t = threading.Thread(target=consumer)
    t.start()
    a = ld.produce_args(1)
    a.gate = GATE_HOST
    a.persistent = 1
    ps = torch.cuda.Stream()
    produce_range(ring, a, 1, 0, n, [0], stream=ps)
    ps.synchronize()
    t.join(60)
    assert not t.is_alive() and len(got) == n
    order = oracle.epoch_order(N, 4, 1)
    for q in range(1, n + 1):
        idx = order[(q - 1) * B:q * B]
        np.testing.assert_array_equal(got[q][1], idx)
        assert got[q][0] == oracle.crc32(oracle.prepare_synthetic(3, 1, idx, 2048 * 4)), q
    a.persistent = 0
    ring.close()


@pytest.mark.parametrize("mode", ["synthetic", "gather"])
def test_persistent_producer_runs_across_epochs(oracle, mode):
    """One persistent launch across epoch boundaries (order_epochs > 1): a
    range that starts mid-epoch and runs through three short epochs of a
    ragged dataset (N % B != 0: each epoch drops its tail, bs/pipeline.py:77-79),
    through a 3-slot ring gated on a host consumer.  Every batch equals the
    oracle's batch of ITS epoch (synthetic: the epoch keys the sample bytes,
    bs/pipeline.py:186; gather: the epoch's own order)."""
    import threading
    import zlib

    from paper_2409_18749_b200._lib import GATE_HOST

    N, B, sb = 1000, 96, 2048  # 10 batches per epoch, 40 samples dropped
    if mode == "synthetic":
        src = SyntheticSource(5, (sb // 4,), DType.I32)
    else:
        src = StoreSource.synthetic(5, N, (sb,))
    ld = CollateLoader(DatasetSpec(src, N, B, shuffle_seed=6))
    L = len(ld)
    assert L == N // B
    ring = DeviceRing(3, ld.batch_nbytes, 1, control="host")
    ring.set_cursor(0, 0)
    e0, b0, n = 2, 7, 2 * L + 5  # epoch 2 batch 7 .. epoch 5 batch 1
    got = {}

    def consumer():
        for q in range(1, n + 1):
            s = ring.slot_of(q)
            ring.host_wait_ready(s, q, timeout_s=60)
            v = ring.view(s, (ld.batch_nbytes,), torch.uint8).cpu().numpy()
            got[q] = (zlib.crc32(v[:ld.input_nbytes].tobytes()),
                      v[ld.input_nbytes:].view(np.int64).copy())
            ring.host_ack(0, q)

    t = threading.Thread(target=consumer)
    t.start()
    k = -(-(b0 + n) // L)
    a = ld.produce_args_epochs(e0, k)
    assert a.order_epochs == k == 4
    a.gate = GATE_HOST
    a.persistent = 1
    ps = torch.cuda.Stream()
    produce_range(ring, a, 1, b0, n, [0], stream=ps)
    ps.synchronize()
    t.join(60)
    assert not t.is_alive() and len(got) == n
    store = None if mode == "synthetic" else oracle.make_store(5, N, sb)
    for q in range(1, n + 1):
        e, bi = divmod(b0 + q - 1, L)
        idx = oracle.epoch_order(N, 6, e0 + e)[bi * B:(bi + 1) * B]
        np.testing.assert_array_equal(got[q][1], idx)
        want = (oracle.prepare_synthetic(5, e0 + e, idx, sb) if mode == "synthetic"
                else oracle.gather(store, idx, sb))
        assert got[q][0] == oracle.crc32(want), q
    ring.close()


def test_multi_epoch_order_is_refused_outside_the_persistent_passthrough():
    """order_epochs > 1 is a persistent-passthrough contract; the per-batch
    producer refuses it loudly instead of reading past the epoch's order."""
    from paper_2409_18749_b200._lib import GATE_HOST

    src = SyntheticSource(5, (512,), DType.I32)
    ld = CollateLoader(DatasetSpec(src, 1000, 96, shuffle_seed=6))
    ring = DeviceRing(3, ld.batch_nbytes, 1, control="host")
    a = ld.produce_args_epochs(0, 2)
    a.gate = GATE_HOST
    a.persistent = 0
    with pytest.raises(Exception, match="multi-epoch"):
        produce_range(ring, a, 1, 0, 12, [0], stream=torch.cuda.Stream())
    ring.close()
