"""Sharded ingest + fused fan-out (tsb_produce_group).

Each writer produces its rows of every batch straight into the same slot of
every ring of the group and publishes its own ready word; a consumer sees a
batch once every writer's shard landed.  On the one-GPU test box the "peer"
rings are distinct allocations on device 0 (in this process, or in other
processes opened over CUDA IPC) -- the same code path as NVLink peers except
for the link.  Parity: every ring's batch equals the oracle's batch
(bit-exact), for the fused collate/augment and the passthrough modes; the
passthrough batches also match the reference's own CRCs (golden)."""

import threading
import zlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2409_18749_b200 import (AugmentSpec, CollateLoader, DatasetSpec,  # noqa: E402
                                   StoreSource, SyntheticSource)
from paper_2409_18749_b200.ring import DeviceRing, produce_group  # noqa: E402
from paper_2409_18749_b200.wire import DType  # noqa: E402


def _run_group(ld, rings, n_shards, epoch, n, expect, writers_map=None):
    """Writers in threads (each blocks on the host gate), one host consumer per
    ring checking every batch with expect(epoch, bi) before releasing it."""
    L = len(ld)
    errors = []

    def consumer(k):
        ring = rings[k]
        try:
            for i in range(n):
                q = epoch * L + 1 + i
                slot = ring.slot_of(q)
                ring.host_wait_ready(slot, q, timeout_s=60)
                got = ring.view(slot, (ld.batch_nbytes,), torch.uint8).cpu().numpy()
                want = expect(epoch, i)
                if got.tobytes() != want.tobytes():
                    bad = np.flatnonzero(got != want)
                    errors.append((k, q, int(bad[0]), len(bad)))
                ring.host_ack(0, q)
        except Exception as e:  # noqa: BLE001
            errors.append((k, repr(e)))
            ring.evict(0)

    def writer(shard, local):
        try:
            s = torch.cuda.Stream()
            a = ld.produce_args(epoch)
            produce_group(rings, local, a, shard, n_shards, epoch * L + 1, 0, n,
                          [[0]] * len(rings), stream=s)
            s.synchronize()
        except Exception as e:  # noqa: BLE001
            errors.append(("writer", shard, repr(e)))

    for r in rings:
        r.set_cursor(0, epoch * L)
    cons = [threading.Thread(target=consumer, args=(k,)) for k in range(len(rings))]
    wrs = [threading.Thread(target=writer, args=(g, (writers_map or {}).get(g, g % len(rings))))
           for g in range(n_shards)]
    for t in cons + wrs:
        t.start()
    for t in cons + wrs:
        t.join(120)
        assert not t.is_alive(), "group pipeline hung"
    assert not errors, errors[:5]


def _expect_augment(oracle, ld, store_h, h, w, c, pad, seed, kind, shuffle_seed, N, B):
    scale, bias = oracle.norm_consts()

    def expect(epoch, bi):
        idx = oracle.epoch_order(N, shuffle_seed, epoch)[bi * B:(bi + 1) * B]
        x = oracle.collate_augment(store_h, idx, h, w, c, pad, True, seed, epoch, kind,
                                   scale if kind else None, bias if kind else None)
        return np.concatenate([x.reshape(-1).view(np.uint8), idx.astype("<i8").view(np.uint8)])

    return expect


@pytest.mark.parametrize("n_shards,n_rings", [(3, 3), (2, 2), (1, 3)])
@pytest.mark.parametrize("out_dtype,kind", [("float32", 1), ("bfloat16", 2), ("uint8", 0)])
def test_group_collate_fanout_parity(oracle, n_shards, n_rings, out_dtype, kind):
    h, w, c, B, N, S, pad = 32, 64, 3, 8, 96, 3, 4
    store = StoreSource.synthetic(6, N, (h, w, c))
    ld = CollateLoader(DatasetSpec(store, N, B, shuffle_seed=4),
                       AugmentSpec(pad=pad, flip=True, out_dtype=out_dtype, seed=3))
    rings = [DeviceRing(S, ld.batch_nbytes, 1, control="host", writers=n_shards)
             for _ in range(n_rings)]
    store_h = oracle.make_store(6, N, h * w * c)
    expect = _expect_augment(oracle, ld, store_h, h, w, c, pad, 3, kind, 4, N, B)
    _run_group(ld, rings, n_shards, 1, 10, expect)
    for r in rings:
        assert r.read_ready(r.slot_of(len(ld) + 10)) == len(ld) + 10
        r.close()


@pytest.mark.parametrize("case_i", [6, 8])  # llm (2048,) i32 B=256; video (16,3,112,112) u8 B=16
@pytest.mark.parametrize("source", ["synthetic", "store"])
def test_group_passthrough_matches_reference_crc(golden, case_i, source):
    case = golden["prepare_batch"][case_i]
    shape, dt = tuple(case["sample_shape"]), DType(case["dtype"])
    N, B = case["samples_per_epoch"], case["batch_size"]
    if source == "synthetic":
        src = SyntheticSource(0, shape, dt)
    else:  # epoch-0 batches of a DirectorySource store == synthetic epoch 0
        src = StoreSource.synthetic(0, N, shape, dt)
    ld = CollateLoader(DatasetSpec(src, N, B, shuffle_seed=0))
    n_shards = 4
    rings = [DeviceRing(2, ld.batch_nbytes, 1, control="host", writers=n_shards)
             for _ in range(2)]
    crcs = {}
    L = len(ld)
    errors = []

    def consumer(k):
        ring = rings[k]
        for i in range(2):
            q = 1 + i
            ring.host_wait_ready(ring.slot_of(q), q, timeout_s=60)
            v = ring.view(ring.slot_of(q), (ld.batch_nbytes,), torch.uint8).cpu().numpy()
            crcs[(k, i)] = zlib.crc32(v[:ld.input_nbytes].tobytes())
            tgt = v[ld.input_nbytes:].view(np.int64)
            if i == 0 and not np.array_equal(tgt, case["indices"]):
                errors.append(("indices", k))
            ring.host_ack(0, q)

    for r in rings:
        r.set_cursor(0, 0)
    cons = [threading.Thread(target=consumer, args=(k,)) for k in range(2)]
    for t in cons:
        t.start()
    ws = []
    for g in range(n_shards):
        def run(g=g):
            s = torch.cuda.Stream()
            produce_group(rings, g % 2, ld.produce_args(0), g, n_shards, 1, 0, 2, [[0], [0]],
                          stream=s)
            s.synchronize()
        ws.append(threading.Thread(target=run))
        ws[-1].start()
    for t in cons + ws:
        t.join(120)
        assert not t.is_alive()
    assert not errors
    assert L >= 2
    assert crcs[(0, 0)] == crcs[(1, 0)] == case["crc32"]
    for r in rings:
        r.close()


def _proc_writer(rank, world, q_out, q_in, res, n):
    """One process per 'GPU' (all on device 0 here): own ring + peers over IPC."""
    import torch

    torch.cuda.set_device(0)
    from oracle import oracle
    from paper_2409_18749_b200 import AugmentSpec, CollateLoader, DatasetSpec, StoreSource
    from paper_2409_18749_b200.ring import DeviceRing, produce_group

    try:
        oracle.load()
        h, w, c, B, N, S = 16, 32, 3, 8, 64, 2
        store = StoreSource.synthetic(1, N, (h, w, c))
        ld = CollateLoader(DatasetSpec(store, N, B, shuffle_seed=7),
                           AugmentSpec(pad=2, flip=True, out_dtype="bfloat16", seed=5))
        own = DeviceRing(S, ld.batch_nbytes, 1, control="host", writers=world)
        own.set_cursor(0, 0)
        q_out.put((rank, own.export(), own.control_name))
        peers = {}
        while len(peers) < world - 1:
            r, hnd, ctl = q_in.get(timeout=120)
            peers[r] = DeviceRing.import_handle(hnd, S, ld.batch_nbytes, 1, ctl, writers=world)
        rings = [own if r == rank else peers[r] for r in range(world)]
        store_h = oracle.make_store(1, N, h * w * c)
        scale, bias = oracle.norm_consts()
        errors = []

        def consume():
            for i in range(n):
                q = 1 + i
                own.host_wait_ready(own.slot_of(q), q, timeout_s=60)
                got = own.view(own.slot_of(q), (ld.batch_nbytes,), torch.uint8).cpu().numpy()
                idx = oracle.epoch_order(N, 7, 0)[i * B:(i + 1) * B]
                x = oracle.collate_augment(store_h, idx, h, w, c, 2, True, 5, 0, 2, scale, bias)
                want = np.concatenate([x.reshape(-1).view(np.uint8),
                                       idx.astype("<i8").view(np.uint8)])
                if got.tobytes() != want.tobytes():
                    errors.append(q)
                own.host_ack(0, q)

        t = threading.Thread(target=consume)
        t.start()
        s = torch.cuda.Stream()
        produce_group(rings, rank, ld.produce_args(0), rank, world, 1, 0, n,
                      [[0]] * world, stream=s)
        s.synchronize()
        t.join(120)
        res.put((rank, "ok" if not errors and not t.is_alive() else f"bad {errors}"))
    except Exception as e:  # noqa: BLE001
        res.put((rank, repr(e)))


def test_group_cross_process_ipc():
    """world=3 writer processes, each owning one ring and writing its shard of
    every batch into all three rings through CUDA-IPC mappings."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    world, n = 3, 8
    qs = [ctx.Queue() for _ in range(world)]
    res = ctx.Queue()
    # route: writer r puts its handle on every other writer's queue
    outs = [ctx.Queue() for _ in range(world)]
    procs = [ctx.Process(target=_proc_writer, args=(r, world, outs[r], qs[r], res, n))
             for r in range(world)]
    for p in procs:
        p.start()
    for r in range(world):  # forward each writer's (handle, control) to the others
        item = outs[r].get(timeout=240)
        for d in range(world):
            if d != r:
                qs[d].put(item)
    results = dict(res.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(60)
    assert results == {r: "ok" for r in range(world)}, results


@pytest.mark.parametrize("out_dtype,kind,checksum", [("float32", 1, False),
                                                    ("bfloat16", 2, False),
                                                    ("float32", 1, True)])
def test_two_stage_input_allgather_then_local_collate(oracle, out_dtype, kind, checksum):
    """Two-stage multi-GPU production: stage 1 all-gathers the compact u8 rows
    into every GPU's input ring (passthrough group, G writers); stage 2 on
    each GPU collates the staged rows into its own output ring
    (tsb_restage_collate).  G = 2 'GPUs' on device 0, threads as ranks."""
    from paper_2409_18749_b200._lib import GATE_HOST
    from paper_2409_18749_b200.collate import _Ingest
    from paper_2409_18749_b200.ring import restage_collate

    h, w, c, B, N, G, n = 32, 64, 3, 8, 64, 2, 12
    store = StoreSource.synthetic(8, N, (h, w, c))
    gather_ld = CollateLoader(DatasetSpec(store, N, B, shuffle_seed=6))
    aug_ld = CollateLoader(DatasetSpec(store, N, B, shuffle_seed=6),
                           AugmentSpec(pad=4, flip=True, out_dtype=out_dtype, seed=2))
    in_rings = [DeviceRing(3, gather_ld.batch_nbytes, 1, control="host", writers=G)
                for _ in range(G)]
    out_rings = [DeviceRing(3, aug_ld.batch_nbytes, 1, control="host") for _ in range(G)]
    for r in in_rings + out_rings:
        r.set_cursor(0, 0)
    tables = [_Ingest(0, B, h * w * c) for _ in range(G)]
    L = len(aug_ld)
    errors, got = [], {g: {} for g in range(G)}
    # checksum: stage 2's collate kernel also writes each output slot's CRC-32
    # (read by the consumer when the slot is published)
    d_crc = [torch.zeros(3, dtype=torch.int32, device="cuda") if checksum else None
             for _ in range(G)]
    crcs = {g: {} for g in range(G)}

    def stage1(g):
        try:
            s = torch.cuda.Stream()
            q = 1
            while q <= n:
                e, bi = divmod(q - 1, L)
                m = min(n - q + 1, L - bi)
                a = gather_ld.produce_args(e)
                produce_group(in_rings, g, a, g, G, q, bi, m, [[0]] * G, stream=s)
                q += m
            s.synchronize()
        except Exception as ex:  # noqa: BLE001
            errors.append(("stage1", g, repr(ex)))

    def stage2(g):
        try:
            s = torch.cuda.Stream()
            q = 1
            while q <= n:
                e, bi = divmod(q - 1, L)
                m = min(n - q + 1, L - bi)
                from paper_2409_18749_b200._lib import ProduceArgs

                base = aug_ld.produce_args(e, with_crc=d_crc[g])
                a = ProduceArgs.from_buffer_copy(base)
                a._keep = base._keep
                a.ingest = tables[g].handle
                a.gate = GATE_HOST
                restage_collate(in_rings[g], 0, out_rings[g], a, q, m, [0], stream=s)
                q += m
            s.synchronize()
        except Exception as ex:  # noqa: BLE001
            errors.append(("stage2", g, repr(ex)))

    def consumer(g):
        r = out_rings[g]
        for q in range(1, n + 1):
            r.host_wait_ready(r.slot_of(q), q, timeout_s=60)
            got[g][q] = r.view(r.slot_of(q), (aug_ld.batch_nbytes,), torch.uint8).cpu().numpy()
            if checksum:
                crcs[g][q] = int(d_crc[g][r.slot_of(q)].item()) & 0xFFFFFFFF
            r.host_ack(0, q)

    ts = [threading.Thread(target=f, args=(g,)) for f in (stage1, stage2, consumer)
          for g in range(G)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(120)
        assert not t.is_alive(), "two-stage pipeline hung"
    assert not errors, errors
    store_h = oracle.make_store(8, N, h * w * c)
    scale, bias = oracle.norm_consts()
    for q in range(1, n + 1):
        e, bi = divmod(q - 1, L)
        idx = oracle.epoch_order(N, 6, e)[bi * B:(bi + 1) * B]
        x = oracle.collate_augment(store_h, idx, h, w, c, 4, True, 2, e, kind, scale, bias)
        want = np.concatenate([x.reshape(-1).view(np.uint8), idx.astype("<i8").view(np.uint8)])
        for g in range(G):
            assert got[g][q].tobytes() == want.tobytes(), (g, q)
            if checksum:
                assert crcs[g][q] == zlib.crc32(want.tobytes()), (g, q)
    for r in in_rings + out_rings:
        r.close()
