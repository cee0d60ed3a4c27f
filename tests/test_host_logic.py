"""Host-side logic of the extensions, on CPU: Join v2 frames, ring
descriptors v2, the heterogeneous-consumer window plan (checked against the
oracle's rebatch indices), shard rows, and the multi-GPU descriptor exchange
over torch.distributed (gloo, world_size 2)."""

import os

import numpy as np
import pytest

from paper_2409_18749_b200 import group
from paper_2409_18749_b200 import segment as sg
from paper_2409_18749_b200.ledger import rebatch_epoch_len, rebatch_window_plan, window_slots
from paper_2409_18749_b200.wire import (DecodeError, EncodeError, Join, PROTOCOL_VERSION, decode,
                                        encode)


def test_join_v1_bytes_unchanged_and_v2_roundtrip():
    assert encode(Join(5)) == bytes.fromhex("0b0000000105000000000000000100")
    m = Join(7, 2, 3, 128)
    assert decode(encode(m)) == m
    assert decode(encode(Join(9, 2))) == Join(9, 2, -1, 0)
    with pytest.raises(EncodeError):
        encode(Join(1, PROTOCOL_VERSION, 0, 0))  # v2 fields need version 2
    bad = bytearray(encode(m))
    bad[13] = 1  # version 1 with a v2-sized body
    with pytest.raises(DecodeError):
        decode(bytes(bad))


def test_ring_descriptor_v1_v2_roundtrip():
    h = bytes(range(64))
    v1 = sg.RingDescriptor(0xABC, 123, 0, 8, 1 << 20, 65, h, "tsbc-1-2")
    assert v1.name().startswith("tsbr:") and sg.RingDescriptor.parse(v1.name()) == v1
    v2 = sg.RingDescriptor(0xABC, 123, 7, 8, 154140672, 65, h, "tsbc-123-abcdef", 8, 256, 16384)
    n = v2.name()
    assert n.startswith("tsbr2:") and len(n) <= 255
    assert sg.RingDescriptor.parse(n) == v2


@pytest.mark.parametrize("P", [32, 64])
@pytest.mark.parametrize("b", [8, 16, 24, 32, 48, 64, 100])
def test_rebatch_plan_yields_reference_batches(oracle, P, b):
    """Walk the consumer's window plan over a simulated stream of producer
    slots: every batch j is exactly order[j*b:(j+1)*b] (the reference's batch
    for size b), a slot is never released while a later window needs it, and
    a window never spans more slots than window_slots() budgets."""
    N = 320
    L = N // P
    order = oracle.epoch_order(N, 11, 2)
    slots = [order[k * P:(k + 1) * P] for k in range(L)]  # producer batch k
    lc = rebatch_epoch_len(N, L, P, b)
    assert lc == min(N, L * P) // b
    released = 0
    for j in range(lc):
        plan = rebatch_window_plan(j, b, P)
        assert plan.k0 >= released, "window needs a released slot"
        assert plan.k1 - plan.k0 + 1 <= window_slots(b, P)
        released = max(released, plan.release_before)
        if plan.zero_copy:
            got = slots[plan.k0][plan.offset:plan.offset + b]
        else:
            got = np.concatenate([slots[k] for k in range(plan.k0, plan.k1 + 1)])[
                plan.offset:plan.offset + b]
            released = max(released, plan.release_after)
        np.testing.assert_array_equal(got, oracle.rebatch_indices(order, b, j))
    assert released <= L


def test_shard_rows_partition_the_batch():
    for b in (8, 9, 256, 257):
        for g in (1, 2, 3, 8):
            if b < g:
                continue
            rows = [group.shard_rows(b, s, g) for s in range(g)]
            assert rows[0][0] == 0 and rows[-1][1] == b
            assert all(rows[i][1] == rows[i + 1][0] for i in range(g - 1))
    with pytest.raises(ValueError):
        group.shard_rows(4, 4, 4)


def _exchange_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        h = bytes([rank]) * 64
        d = sg.RingDescriptor(rank, os.getpid(), rank, 8, 4096, 5, h, f"tsbc-{rank}", world,
                              256, 16384)
        got = group.exchange(d)
        q.put((rank, [(x.ring_id, x.device, x.ipc_handle[0], x.writers) for x in got]))
    finally:
        dist.destroy_process_group()


def test_descriptor_exchange_gloo_world2():
    import multiprocessing as mp
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_exchange_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(30)
    want = [(0, 0, 0, 2), (1, 1, 1, 2)]
    assert res == {0: want, 1: want}


def test_connect_error_when_no_producer(tmp_path):
    """No producer at the endpoints: the consumer fails with StreamError after
    its connect timeout (pkg/tests/test_producer_consumer.py:436-445)."""
    from paper_2409_18749_b200 import SharedLoader
    from paper_2409_18749_b200.errors import StreamError

    ld = SharedLoader(f"unix:{tmp_path}/nope-b.sock", f"unix:{tmp_path}/nope-a.sock",
                      consumer_id=1, connect_timeout_s=0.3)
    with pytest.raises(StreamError):
        next(iter(ld))


def test_consumer_heartbeat_cadence(tmp_path):
    """A scripted producer (raw sockets, the wire codec) admits one
    SharedLoader and times its Heartbeats on the aggregate channel: ~10 in
    1.1 s at a 100 ms interval, no gap above 2x the interval plus slack
    (pkg/tests/test_producer_consumer.py:518-556)."""
    import socket
    import threading
    import time

    from paper_2409_18749_b200 import SharedLoader
    from paper_2409_18749_b200.transport import listen
    from paper_2409_18749_b200.wire import FrameDecoder, Heartbeat, Join, Welcome, encode

    b_ep, a_ep = f"unix:{tmp_path}/fb.sock", f"unix:{tmp_path}/fa.sock"
    lb, la = listen(b_ep), listen(a_ep)
    box = {}

    def client():
        ld = SharedLoader(b_ep, a_ep, consumer_id=6, heartbeat_interval_s=0.1, device=0)
        ld._connect()
        box["ld"] = ld
        time.sleep(1.1)
        ld.finished = True

    t = threading.Thread(target=client)
    t.start()
    bs, _ = lb.accept()
    bs.recv(4096)  # identification heartbeat
    ag, _ = la.accept()
    dec = FrameDecoder()
    while not any(isinstance(m, Join) for m in dec.feed(ag.recv(4096))):
        pass
    ag.sendall(encode(Welcome(6, 0, 10, 0, 2, 2)))
    ag.settimeout(3.0)
    arrivals = []
    deadline = time.monotonic() + 1.2
    while time.monotonic() < deadline:
        try:
            data = ag.recv(4096)
        except socket.timeout:
            break
        if not data:
            break
        arrivals += [time.monotonic() for m in dec.feed(data) if isinstance(m, Heartbeat)]
    t.join(10)
    for s in (bs, ag, lb, la):
        s.close()
    assert len(arrivals) >= 8
    assert max(b - a for a, b in zip(arrivals, arrivals[1:])) < 0.25
