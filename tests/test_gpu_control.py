"""Control-plane parity on the device ring: the
reference's integration tests (pkg/tests/test_producer_consumer.py:231-414)
re-run against the B200 facade -- backpressure / drift bound, eviction that
unblocks survivors (cursor sentinel), rubberband replay from retained ring
slots, late join waiting for the next epoch, and exactly-once in-order
delivery."""

import threading
import time

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2409_18749_b200 import SharedLoader, TensorProducer  # noqa: E402


class SeqLoader:
    """(input, target) batches whose target carries the global batch number."""

    def __init__(self, n, batch=4, delay_s=0.0):
        self.n, self.batch, self.delay_s = n, batch, delay_s  # delay_s: simulated prep cost
        self.epoch = 0

    def __len__(self):
        return self.n

    def __iter__(self):
        e = self.epoch
        self.epoch += 1
        for i in range(self.n):
            if self.delay_s:
                time.sleep(self.delay_s)
            inp = np.full((self.batch, 16), e * 1000 + i, dtype=np.float32)
            yield inp, np.array([e, i] + [0] * (self.batch - 2), dtype=np.int64)


def expected(epochs, n, start_epoch=0):
    return [(e, i) for e in range(start_epoch, epochs) for i in range(n)]


@pytest.fixture
def endpoints(tmp_path):
    return f"unix:{tmp_path}/cb.sock", f"unix:{tmp_path}/ca.sock"


def run_producer(loader, endpoints, epochs, **kw):
    b, a = endpoints
    producer = TensorProducer(loader, broadcast=b, aggregate=a, **kw)

    def run():
        for _ in range(epochs):
            for _ in producer:
                pass
        producer.join(20)

    t = threading.Thread(target=run, daemon=True)
    t.start()
    return producer, t


def consume(endpoints, cid, epochs, out, delay_s=0.0, stop_after=None, **kw):
    loader = SharedLoader(*endpoints, consumer_id=cid, **kw)
    out["loader"] = loader
    seq = out.setdefault("seq", [])
    with torch.cuda.stream(torch.cuda.Stream()):
        for _ in range(epochs):
            for inp, tgt in loader:
                t = tgt.cpu().numpy()
                v = float(inp[0, 0].item())
                assert v == t[0] * 1000 + t[1]  # input paired with its own target
                seq.append((int(t[0]), int(t[1])))
                if delay_s:
                    time.sleep(delay_s)
                if stop_after is not None and len(seq) >= stop_after:
                    return  # stalled: stops fetching (holds its slot) ...
            if loader.finished:
                break
    loader.close()


def test_slow_consumer_backpressure(endpoints):
    """Flow gate (bs/producer.py:230-238, sl/producer.py:291-294): the producer
    announces only while fewer than buffer_depth batches await the slowest
    consumer's ack -- extra ring slots serve retention and rebatching, not
    run-ahead (pkg/tests/test_producer_consumer.py:273-288)."""
    producer, pt = run_producer(SeqLoader(12), endpoints, 1, buffer_depth=2, ring_slots=8)
    out = {}
    w = threading.Thread(target=consume, args=(endpoints, 1, 1, out), kwargs={"delay_s": 0.05})
    w.start()
    for _ in range(6):
        time.sleep(0.07)
        announced = producer.stats["announced"]
        fetched = out["loader"].fetched if "loader" in out else 0
        assert announced <= fetched + 2
    w.join(30)
    pt.join(30)
    assert out["seq"] == expected(1, 12)
    producer.close()


@pytest.mark.parametrize("depth", [1, 2, 3])
def test_drift_bound_mixed_speeds(endpoints, depth):
    """SPEC.md:524 criterion 4: over the whole run, max - min wire-ack cursor
    across admitted consumers stays <= buffer_depth (ledger drift series), for
    consumers of very different speeds; and SPEC.md:528 criterion 8: at most
    N+1 slots are live (announced, not yet released by every consumer) when
    no rubberband window is open."""
    E, n = 2, 24
    producer, pt = run_producer(SeqLoader(n), endpoints, E, buffer_depth=depth, ring_slots=8,
                                min_consumers=3)
    outs = [{} for _ in range(3)]
    ts = [threading.Thread(target=consume, args=(endpoints, 20 + k, E, outs[k]),
                           kwargs={"delay_s": d}) for k, d in enumerate((0.0, 0.004, 0.02))]
    for t in ts:
        t.start()
    for t in ts:
        t.join(120)
    pt.join(60)
    for o in outs:
        assert o["seq"] == expected(E, n)
    assert producer._ledger.drift_series, "no drift samples"
    assert producer._ledger.drift_max <= depth, producer._ledger.drift_series
    assert 1 <= producer.stats["live_max"] <= depth + 1
    producer.close()


def test_checksum_exactly_once_three_consumers(endpoints):
    """SPEC.md:525 criterion 5 with checksums on (bs/harness.py:636-671): each
    consumer's (epoch, index, checksum) sequence equals the producer's records,
    zero duplicates; every announced checksum is the zlib CRC-32 of the bytes
    the consumer actually read (input bytes + target bytes, the pair ABI);
    one consumer also verifies on the device (verify_checksum)."""
    import zlib

    E, n = 2, 10
    producer, pt = run_producer(SeqLoader(n), endpoints, E, min_consumers=3, checksum=True)
    outs = [{} for _ in range(3)]

    def run(k):
        o = outs[k]
        loader = SharedLoader(*endpoints, consumer_id=40 + k, verify_checksum=(k == 0))
        recs = o.setdefault("recs", [])
        with torch.cuda.stream(torch.cuda.Stream()):
            for _ in range(E):
                for inp, tgt in loader:
                    a = loader.last_announce
                    raw = inp.cpu().numpy().tobytes() + tgt.cpu().numpy().tobytes()
                    assert zlib.crc32(raw) == a.checksum
                    recs.append((a.epoch, a.batch_index, a.checksum))
                if loader.finished:
                    break
        loader.close()

    ts = [threading.Thread(target=run, args=(k,)) for k in range(3)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(120)
    pt.join(60)
    assert len(producer.batches) == E * n
    assert all(c != 0 for _, _, c in producer.batches)
    for o in outs:
        assert o["recs"] == producer.batches
    producer.close()


def test_exactly_once_in_order_three_consumers_two_epochs(endpoints):
    producer, pt = run_producer(SeqLoader(20), endpoints, 2, min_consumers=3, ring_slots=4)
    outs = [{} for _ in range(3)]
    ts = [threading.Thread(target=consume, args=(endpoints, 10 + k, 2, outs[k]))
          for k in range(3)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(60)
    pt.join(30)
    for o in outs:
        assert o["seq"] == expected(2, 20)
    assert producer.stats["announced"] == 40
    producer.close()


def test_eviction_unblocks_survivors(endpoints):
    """Criterion 7: a consumer that stops fetching and heartbeating is evicted
    after the timeout; its cursor becomes the sentinel, so the device ring
    stops waiting for it and the survivor gets every batch."""
    producer, pt = run_producer(SeqLoader(40), endpoints, 1, min_consumers=2, ring_slots=4,
                                heartbeat_timeout_s=0.5)
    victim, survivor = {}, {}

    def run_victim():
        consume(endpoints, 2, 1, victim, stop_after=3, heartbeat_interval_s=0.1)
        victim["loader"].finished = True  # heartbeats stop too (process "hung")

    vt = threading.Thread(target=run_victim)
    st = threading.Thread(target=consume, args=(endpoints, 1, 1, survivor),
                          kwargs={"heartbeat_interval_s": 0.1})
    vt.start()
    st.start()
    vt.join(30)
    st.join(60)
    pt.join(60)
    assert producer.stats["evictions"] == 1
    assert survivor["seq"] == expected(1, 40)
    assert victim["seq"] == expected(1, 40)[:3]
    producer.close()


def test_rubberband_replay_race_no_delays(endpoints):
    """A rubberband joiner whose broadcast announces overtake its private
    replay (no loader or consumer delays) still gets the whole epoch in order:
    overtaking announces wait for the replayed prefix instead of being dropped
    (bs/producer.py:599-685 halts; here the flow gate holds the producer on the
    joiner's cursor and the consumer buffers the overtakers)."""
    for trial in range(3):
        b, a = endpoints
        eps = (b + f".{trial}", a + f".{trial}")
        producer, pt = run_producer(SeqLoader(32), eps, 2, rubberband_fraction=0.25,
                                    ring_slots=16, buffer_depth=2)
        base, joiner = {}, {}
        gate = threading.Event()

        def run_base():
            loader = SharedLoader(*eps, consumer_id=1)
            base["loader"] = loader
            seq = base.setdefault("seq", [])
            with torch.cuda.stream(torch.cuda.Stream()):
                for _ in range(2):
                    for inp, tgt in loader:
                        t = tgt.cpu().numpy()
                        seq.append((int(t[0]), int(t[1])))
                        if len(seq) == 1:
                            gate.wait(30)  # hold the producer inside the window
                    if loader.finished:
                        break
            loader.close()

        bt = threading.Thread(target=run_base)
        bt.start()
        deadline = time.time() + 30
        while producer.stats["announced"] < 2 and time.time() < deadline:
            time.sleep(0.001)
        jt = threading.Thread(target=consume, args=(eps, 2, 2, joiner))
        jt.start()
        deadline = time.time() + 30
        while "loader" not in joiner and time.time() < deadline:
            time.sleep(0.001)
        while joiner["loader"].welcome is None and time.time() < deadline:
            time.sleep(0.001)
        gate.set()
        jt.join(60)
        bt.join(60)
        pt.join(60)
        assert joiner["loader"].welcome.admitted == 1  # ADMIT_RUBBERBAND
        assert base["seq"] == expected(2, 32)
        assert joiner["seq"] == expected(2, 32)
        producer.close()


def test_rubberband_join_gets_full_epoch(endpoints):
    """A consumer joining inside the rubberband window (fraction of the epoch)
    is admitted at once and replayed the retained slots from the ring: it
    sees the full epoch, then keeps streaming the next one."""
    producer, pt = run_producer(SeqLoader(16, delay_s=0.05), endpoints, 2,
                                rubberband_fraction=0.25, ring_slots=8)
    base, joiner = {}, {}
    bt = threading.Thread(target=consume, args=(endpoints, 1, 2, base), kwargs={"delay_s": 0.02})
    bt.start()
    deadline = time.time() + 30
    while producer.stats["announced"] < 2 and time.time() < deadline:
        time.sleep(0.002)
    assert producer.stats["announced"] < 4  # still inside the window of ceil(0.25*16) = 4
    consume(endpoints, 2, 2, joiner)
    bt.join(60)
    pt.join(60)
    assert base["seq"] == expected(2, 16)
    assert joiner["seq"] == expected(2, 16)
    assert joiner["loader"].welcome.admitted == 1  # ADMIT_RUBBERBAND
    producer.close()


def test_late_join_waits_for_next_epoch(endpoints):
    producer, pt = run_producer(SeqLoader(20), endpoints, 2, rubberband_fraction=0.05,
                                ring_slots=4)
    base, joiner = {}, {}
    bt = threading.Thread(target=consume, args=(endpoints, 1, 2, base), kwargs={"delay_s": 0.01})
    bt.start()
    deadline = time.time() + 30
    while producer.stats["announced"] < 6 and time.time() < deadline:
        time.sleep(0.002)
    consume(endpoints, 2, 1, joiner)
    bt.join(60)
    pt.join(60)
    assert base["seq"] == expected(2, 20)
    assert joiner["seq"] == expected(2, 20, start_epoch=1)
    assert joiner["loader"].welcome.admitted == 0  # ADMIT_WAIT
    producer.close()


def test_consumer_churn_reuses_cursor_words(endpoints):
    """More consumers over a job's life than cursor words: a departed
    consumer's word (Bye) is reused after the quarantine, so a long-running
    producer keeps admitting newcomers.  An anchor consumer stays for the
    whole run (with no admitted consumer the producer pauses, as the
    reference's does, sl/producer.py:282-285); five newcomers in turn share
    the one remaining word, each receiving one whole epoch."""
    E = 100
    producer, pt = run_producer(SeqLoader(8, delay_s=0.01), endpoints, E, ring_slots=4,
                                max_consumers=2, heartbeat_timeout_s=0.25)
    anchor = {}
    at = threading.Thread(target=consume, args=(endpoints, 1, E, anchor),
                          kwargs={"heartbeat_interval_s": 0.05})
    at.start()
    deadline = time.time() + 30
    while producer.stats["announced"] < 1 and time.time() < deadline:
        time.sleep(0.002)
    cursors = []
    for k in range(5):
        out = {}
        consume(endpoints, 100 + k, 1, out, heartbeat_interval_s=0.05)
        cursors.append(out["loader"]._cursor)
        e0 = out["seq"][0][0]
        assert out["seq"] == [(e0, i) for i in range(8)]  # one whole epoch, in order
        time.sleep(producer.cursor_quarantine_s + 0.1)
    assert cursors == [1] * 5 and anchor["loader"]._cursor == 0  # 6 consumers on 2 words
    assert len(producer.drops) == 5 and all(d[1] in ("bye", "disconnect") for d in producer.drops)
    at.join(60)
    pt.join(60)
    assert anchor["seq"] == expected(E, 8)
    producer.close()


def test_zero_consumers_idle(endpoints):
    """With no consumer the producer announces nothing (it waits at the start
    barrier); a consumer that arrives later gets the whole epoch
    (pkg/tests/test_producer_consumer.py:290-298)."""
    producer, pt = run_producer(SeqLoader(5), endpoints, 1)
    time.sleep(0.5)
    assert producer.stats["announced"] == 0
    out = {}
    consume(endpoints, 1, 1, out)
    pt.join(30)
    assert out["seq"] == expected(1, 5)
    producer.close()


def test_all_consumers_evicted_producer_pauses(endpoints):
    """The only consumer stops heartbeating and is evicted: the producer then
    announces nothing more until someone is admitted again
    (pkg/tests/test_producer_consumer.py:336-365)."""
    producer, pt = run_producer(SeqLoader(200), endpoints, 1, ring_slots=4,
                                heartbeat_timeout_s=0.4)
    victim = {}
    consume(endpoints, 1, 1, victim, stop_after=2, heartbeat_interval_s=0.1)
    victim["loader"].finished = True  # heartbeats stop ("hung")
    deadline = time.time() + 10
    while producer.stats["evictions"] < 1 and time.time() < deadline:
        time.sleep(0.01)
    assert producer.stats["evictions"] == 1
    time.sleep(0.3)
    a = producer.stats["announced"]
    time.sleep(0.5)
    assert producer.stats["announced"] == a < 200  # paused with no consumers
    producer.join(0.0)
    pt.join(30)
    producer.close()


def test_version_mismatch_drops_connection(endpoints):
    """A Join with an unknown protocol version is closed without a Welcome;
    the producer keeps serving (pkg/tests/test_producer_consumer.py:418-434)."""
    from paper_2409_18749_b200.transport import dial
    from paper_2409_18749_b200.wire import Heartbeat, encode

    producer, pt = run_producer(SeqLoader(5), endpoints, 1)
    b, a = endpoints
    bs = dial(b, 5)
    bs.sendall(encode(Heartbeat(9, 0)))
    ag = dial(a, 5)
    ag.sendall(bytes.fromhex("0b000000" "01" "0900000000000000" "6300"))  # Join(9, version 99)
    ag.settimeout(10)
    assert ag.recv(4096) == b""
    bs.close()
    ag.close()
    out = {}
    consume(endpoints, 1, 1, out)
    pt.join(30)
    assert out["seq"] == expected(1, 5)
    assert 9 not in [d[0] for d in producer.drops]  # never admitted
    producer.close()
