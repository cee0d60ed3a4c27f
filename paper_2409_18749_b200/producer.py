"""TensorProducer: the producer half of the drop-in pair (sl/producer.py:43-337).

Usage is the reference's (Listing 1b)::

    producer = TensorProducer(data_loader)
    for epoch in range(epochs):
        for _ in producer:        # one pass over the wrapped loader
            pass
    producer.join()

Differences behind the same API (B200 data plane):

* batches live in a device-HBM ring (``DeviceRing``) instead of one POSIX shm
  segment per batch; a ``CollateLoader`` writes each batch straight into its
  slot with the fused collate/augment kernel, any other loader's (input,
  target) pairs are copied in once;
* release is counted in cursor words: consumers advance their cursor (from
  their own CUDA stream, or a host store into the host-shared control block);
  before reusing a slot the producer thread checks the cursors on the host
  (control="host": the producer's streams never wait on a device word) or its
  stream waits on them (control="device"); the Ack frames still feed the
  reference's ledger bookkeeping;
* the reference's wire protocol is kept byte-for-byte (Join/Welcome/Announce/
  Ack/Heartbeat/EpochStart/EpochEnd/Bye/Shutdown); the Announce's segment
  name carries the slot and its 80-byte segment header (segment.py).

Keyword-only extensions: ``ring_slots`` (device ring depth; bounds drift),
``control`` ("host": ring control words in a host-shared, device-mapped
shm block -- evictions and map-and-ack consumers never touch a GPU channel;
"device": words in HBM), ``min_consumers`` (start barrier, bs/producer.py:73-76 -- the facade's
missing barrier is the start race noted in SURVEY.md §4), ``checksum``
(device CRC-32 of every batch into Announce.checksum; default on for one GPU,
as the reference checksums every segment), ``rubberband_fraction``
(late-join replay window, bs/producer.py:119-135; 0 = facade behaviour),
``device``; ``devices`` + ``fanout`` (multi-GPU, below).

Multi-GPU (``devices=[0, 1, ...]``): one ring per device, each
consumer maps the ring of its own GPU (``SharedLoader(device=...)``, Join v2).
``fanout="auto"`` (default) picks ``"inputs"`` for an augmenting
``CollateLoader`` and ``"sharded"`` otherwise.  ``fanout="sharded"``: every
device collates its 1/G rows of each
batch and the kernel stores them into the same slot of every device's ring
(P2P stores over NVLink/NVSwitch -- the all-gather fused into the producing
kernel, ``tsb_produce_group``); ``fanout="inputs"`` (two-stage): every
device gathers its 1/G compact u8 rows into every device's input ring, then
each device collates the whole batch locally (a quarter of the NVLink bytes
at f32); ``fanout="star"``: the first device produces the
whole batch into every ring (the literal single-producer fan-out).

Heterogeneous consumers (``SharedLoader(batch_size=b)``): each receives
exactly the reference's batches for its own batch size -- samples
``order[j*b:(j+1)*b]`` of the batch-size-independent epoch order
(bs/pipeline.py:113-123), drop-last ``N // b`` -- as zero-copy windows of the
producer's slots, or gathered by the rebatch kernel when a window straddles
two slots.
"""

from __future__ import annotations

import collections
import os
import threading
import time
from collections import deque

import numpy as np

from . import dataplane as dp
from . import segment as sg
from .errors import ProducerClosed
from .ledger import (ConsumerRecord, Ledger, admission_code, rebatch_epoch_len, retention_window,
                     seq_of, window_slots)
from ._lib import GATE_HOST
from .ring import DeviceRing, produce_group_multi, produce_range, restage_collate
from .hub import Hub
from .transport import HANDOFF, Conn, endpoints_from_env, listen
from .wire import (ADMIT_IMMEDIATE, ADMIT_RUBBERBAND, ADMIT_WAIT, SUPPORTED_VERSIONS, Ack,
                   Announce, Bye, DType, EpochEnd, EpochStart, Heartbeat, Join, Shutdown, Welcome,
                   dtype_of, encode)

MONITOR_ID = 0  # bs/producer.py:52-54: passive broadcast observers
SENTINEL_MIN = 1 << 61  # cursors at or above this are evicted / unused words
_RINGS: dict[int, DeviceRing] = {}  # ring_id -> ring, for same-process consumers


def local_ring(ring_id: int):
    return _RINGS.get(ring_id)


ANN_LAG = int(os.environ.get("TSB_ANN_LAG", "2"))
# fast path with a checksum: Announce this many launches behind (1 keeps the host
# in lockstep with the GPU: each launch then waits for the previous batch); the
# ack gate bounds it by buffer_depth


class TensorProducer:
    def __init__(self, data_loader, broadcast: str | None = None, aggregate: str | None = None,
                 buffer_depth: int = 2, heartbeat_timeout_s: float = 5.0,
                 pause_poll_s: float = 0.05, *, ring_slots: int | None = None,
                 min_consumers: int = 1, checksum: bool | None = None,
                 rubberband_fraction: float = 0.0, max_consumers: int = 64,
                 device: int | None = None, control: str = "host", devices=None,
                 fanout: str = "auto"):
        import torch

        if not hasattr(data_loader, "__len__"):
            raise TypeError("data_loader must have a length (batches per epoch)")
        if buffer_depth < 1 or min_consumers < 1:
            raise ValueError("buffer_depth and min_consumers must be >= 1")
        if not 0 <= rubberband_fraction < 1:
            raise ValueError("rubberband_fraction must be in [0, 1)")
        self._loader = data_loader
        self._device_loader = hasattr(data_loader, "produce_into")
        self._broadcast_ep, self._aggregate_ep = endpoints_from_env(broadcast, aggregate)
        self._depth = buffer_depth
        self._hb_timeout = heartbeat_timeout_s
        self._poll = pause_poll_s
        self._min_consumers = min_consumers
        self._checksum_arg = checksum
        self._fraction = rubberband_fraction
        self._max_consumers = max_consumers
        self._ring_slots = ring_slots
        self._control = control
        self.device = torch.cuda.current_device() if device is None else device
        self._devices = [int(d) for d in devices] if devices else [self.device]
        if not 1 <= len(self._devices) <= 8:
            raise ValueError("1..8 devices")
        self.device = self._devices[0]
        if fanout not in ("auto", "sharded", "star", "inputs"):
            raise ValueError("fanout must be 'auto', 'sharded', 'star' or 'inputs'")
        if fanout == "auto":  # two-stage where a collate follows the gather, else sharded
            fanout = "inputs" if (getattr(data_loader, "augment", None) is not None and
                                  hasattr(data_loader, "dataset")) else "sharded"
        self.fanout = fanout
        self._multi = len(self._devices) > 1
        # every batch's CRC-32 rides in its Announce, as the reference's
        # create_segment computes it (bs/payload.py:218, sl/producer.py:313):
        # the default on one GPU; the fused multi-GPU fan-out paths announce 0
        # (no checksum) unless checksum=True selects the per-device path
        self._checksum = (not self._multi) if checksum is None else bool(checksum)
        if self._multi and control != "host":
            raise ValueError("multi-GPU rings need control='host' (host-shared control words)")
        self._sharded = self._multi and fanout == "sharded"
        # two-stage: every device gathers its 1/G u8 rows of each
        # batch into every device's input ring, then each device collates the
        # whole staged batch into its own ring
        self._two_stage = self._multi and fanout == "inputs"
        if self._two_stage and not (getattr(data_loader, "augment", None) is not None and
                                    hasattr(data_loader, "dataset")):
            raise ValueError("fanout='inputs' needs a CollateLoader with an AugmentSpec")
        self._in_rings: dict[int, DeviceRing] = {}
        self._streams2: dict = {}
        self._tables: dict = {}
        self._gather_loader = None
        self._chain2_ok = False
        self._rings: dict[int, DeviceRing] = {}
        self._streams: dict = {}
        self._descriptors: dict[int, sg.RingDescriptor] = {}
        self._ring_ids: dict[int, int] = {}
        self._orders: dict = {}
        self._per_slot = 0   # producer batch size (samples per slot)
        self._samples = 0    # samples per epoch
        self._epoch = 0
        self._announced_in_epoch = 0
        self._epoch_started = False
        self._barrier_met = False
        self._lock = threading.Condition()
        self._consumers: dict[int, ConsumerRecord] = {}
        self._bcast_pending: dict[int, Conn] = {}
        self._monitors: list[Conn] = []
        self._ledger = Ledger()
        self._next_cursor = 0
        # cursor words of departed consumers, reused after a quarantine: a
        # consumer that left (Bye, closed socket, rejoin) may still have one ack
        # store in flight.  Timed-out consumers' words are never reused -- a hung
        # process can wake up and store its old cursor (bs/producer.py:203-219
        # evicts; here the word stays the eviction sentinel for good).
        self._free_cursors: deque = deque()  # (cursor, free time)
        self._closed = False
        self._started = False
        self._listeners = []
        self._threads: list[threading.Thread] = []
        self._ring: DeviceRing | None = None
        self._stream = None
        self._events = []
        self._retained: dict[int, dict] = {}  # seq -> {device: announce} (rubberband prefix)
        self._retention_active = False
        self.ring_id = (os.getpid() << 20) ^ (id(self) & 0xFFFFF)
        self.stats = {"announced": 0, "acks": 0, "evictions": 0, "live_max": 0,
                      "live_max_window": 0}
        # (epoch, batch_index, checksum) of every announced batch, the
        # reference's RunReport.batches (bs/producer.py:528) for exactly-once checks
        self.batches: list[tuple[int, int, int]] = []
        self.drops: list[tuple[int, str, float]] = []  # (consumer_id, reason, time) event log
        self._chain_ok = False  # PDL across produce calls (previous op = our fused kernel)
        # wire Acks are queued by the reader threads without taking the lock and
        # folded into the ledger in bulk by the producer (_drain_acks): one lock
        # round and one drift sample per batch instead of per ack
        self._ack_q: deque = deque()
        # native control-plane hub: admitted consumers' aggregate sockets are read
        # (Acks, Heartbeats, Bye) and Announces written without the interpreter
        self._hub = Hub()
        self._hub_fds: dict[int, int] = {}  # fd -> consumer id
        self._hdr_key = None
        self._hdr_reserved = b""
        # checksum=True: a batch is announced once its CRC-32 reached the host,
        # which is after the NEXT batch was enqueued (the ingest / collate
        # of batch q+1 never waits for batch q's checksum)
        self._pending_ann = None
        # the fast path with a checksum announces ANN_LAG batches behind the
        # launch: the batch's CRC (stored by the kernel) is then already there
        self._pend_fast = collections.deque()
        self._settled = None  # (announce, result) awaiting bookkeeping (split fast path)
        self._live_lists = None  # the host gate's live cursors (live-slot sampling)
        # the one-GPU device-loader fast path (hub.Facade): consumer lists are
        # pushed to it when _cver (bumped on every membership change) moves
        self._cver = 0
        self._facade = None
        self._facade_ver = -1
        self._facade_epoch = None
        self._facade_fds: dict = {}
        self._since_drain = 0

    # -- ring -------------------------------------------------------------
    def _batch_nbytes_hint(self) -> int | None:
        return getattr(self._loader, "batch_nbytes", None)

    def _ensure_ring(self, nbytes: int) -> None:
        import torch

        if self._ring is not None:
            if nbytes > self._ring.slot_bytes:
                raise ValueError(f"batch of {nbytes} B exceeds the ring slot "
                                 f"({self._ring.slot_bytes} B); batch shapes must be fixed")
            return
        window = retention_window(self._fraction, max(1, len(self._loader)))
        slots = self._ring_slots or max(self._depth + 2 + window, 4)
        if slots <= window:
            raise ValueError(f"ring_slots={slots} must exceed the rubberband window {window}")
        if self._multi:
            from . import dataplane as dp

            for a in set(self._devices):  # kernels on a store into (and read from) b over NVLink
                for b in set(self._devices):
                    if a != b:
                        if not dp.can_access_peer(a, b):
                            raise ValueError(f"GPU {a} cannot access GPU {b} (no P2P)")
                        dp.enable_peer(a, b)
        writers = len(self._devices) if self._sharded else 1  # two-stage: one writer per ring
        for k, d in enumerate(self._devices):
            with torch.cuda.device(d):
                # cursor index max_consumers is the producer's retention cursor
                ring = DeviceRing(slots, nbytes, self._max_consumers + 1, device=d,
                                  control=self._control, writers=writers)
                self._rings[k] = ring
                self._streams[k] = torch.cuda.Stream(device=d)
                rid = self.ring_id if k == 0 else (self.ring_id ^ (k << 44))
                self._ring_ids[k] = rid
                _RINGS[rid] = ring
        if self._two_stage:
            from .collate import CollateLoader, _Ingest

            ds = self._loader.dataset
            self._gather_loader = CollateLoader(ds)  # u8 rows + target indices (stage 1)
            for k, d in enumerate(self._devices):
                with torch.cuda.device(d):
                    r = DeviceRing(4, self._gather_loader.batch_nbytes, 1, device=d,
                                   control="host", writers=len(self._devices))
                    r.set_cursor(0, 0)
                    self._in_rings[k] = r
                    self._streams2[k] = torch.cuda.Stream(device=d)
                    self._tables[k] = _Ingest(d, ds.batch_size, ds.source.sample_nbytes)
        self._ring = self._rings[0]
        self._stream = self._streams[0]
        with torch.cuda.device(self.device):
            self._events = [torch.cuda.Event() for _ in range(slots)]
            for e in self._events:  # materialise the CUDA events (native code records them)
                e.record(self._stream)
            self._crc = torch.zeros(slots, dtype=torch.int32, device=f"cuda:{self.device}")
            self._crc_host = torch.zeros(slots, dtype=torch.int32).pin_memory()
        self._lock.notify_all()

    def _descriptor_for(self, k: int) -> sg.RingDescriptor:
        """Ring k (on self._devices[k]) as a consumer maps it."""
        if k not in self._descriptors:
            ring = self._rings[k]
            self._descriptors[k] = sg.RingDescriptor(
                self._ring_ids[k], os.getpid(), self._devices[k], ring.slots, ring.slot_bytes,
                self._max_consumers + 1, ring.export(), ring.control_name, ring.writers,
                self._per_slot, self._samples)
        return self._descriptors[k]

    def _ring_for_device(self, dev: int) -> int | None:
        """Ring index serving a consumer on `dev` (least loaded if several)."""
        ks = [k for k, d in enumerate(self._devices) if d == dev]
        if not ks:
            return None
        load = {k: sum(1 for r in self._consumers.values() if r.ring == k) for k in ks}
        return min(ks, key=lambda k: (load[k], k))

    @property
    def ring(self) -> DeviceRing | None:
        return self._ring

    @property
    def rings(self) -> dict:
        return dict(self._rings)

    def _set_geometry(self, first_batch=None) -> None:
        """Producer batch size and samples per epoch (rebatch descriptors)."""
        if self._per_slot:
            return
        ds = getattr(self._loader, "dataset", None)
        if ds is not None and hasattr(ds, "batch_size"):
            self._per_slot = int(ds.batch_size)
            self._samples = int(getattr(ds, "samples_per_epoch", 0))
        elif first_batch is not None:
            shape = getattr(first_batch[0], "shape", ())
            self._per_slot = int(shape[0]) if len(shape) else 1
            self._samples = self._per_slot * len(self._loader)

    def _rebatch_ok(self, b: int) -> bool:
        """A consumer batch size is servable when the drop-last epoch has a
        batch of it and a window fits the ring next to the producer's run-ahead."""
        if not self._per_slot or b <= 0:
            return False
        L = max(1, len(self._loader))
        if rebatch_epoch_len(self._samples, L, self._per_slot, b) < 1:
            return False
        return window_slots(b, self._per_slot) + 1 <= self._ring.slots

    @property
    def _retention_cursor(self) -> int:
        return self._max_consumers

    # -- server plumbing --------------------------------------------------
    def _start(self) -> None:
        if self._started:
            return
        self._started = True
        self._hub.set_epoch_len(max(1, len(self._loader)))
        hint = self._batch_nbytes_hint()
        if hint is not None:
            with self._lock:
                self._set_geometry()
                self._ensure_ring(hint)
        for ep, handler in ((self._broadcast_ep, self._accept_broadcast),
                            (self._aggregate_ep, self._accept_aggregate)):
            lst = listen(ep)
            self._listeners.append(lst)
            t = threading.Thread(target=handler, args=(lst,), daemon=True)
            t.start()
            self._threads.append(t)
        t = threading.Thread(target=self._sweep_loop, daemon=True)
        t.start()
        self._threads.append(t)

    def _accept_broadcast(self, lst) -> None:
        while True:
            try:
                sock, _ = lst.accept()
            except OSError:
                return
            conn = Conn(sock)
            state = {"cid": None}

            def on_msg(m, conn=conn, state=state):
                if state["cid"] is None and isinstance(m, Heartbeat):
                    state["cid"] = m.consumer_id
                    with self._lock:
                        if m.consumer_id == MONITOR_ID:
                            self._monitors.append(conn)
                        elif m.consumer_id in self._consumers:
                            self._consumers[m.consumer_id].bcast = conn
                        else:
                            self._bcast_pending[m.consumer_id] = conn
                        self._cver += 1
                        self._lock.notify_all()

            def on_close(conn=conn, state=state):
                with self._lock:
                    cid = state["cid"]
                    if cid == MONITOR_ID and conn in self._monitors:
                        self._monitors.remove(conn)
                        self._cver += 1
                    elif cid is not None and cid in self._consumers and \
                            self._consumers[cid].bcast is conn:
                        self._drop(cid, "disconnect")

            conn.start_reader(on_msg, on_close, "bcast-reader")

    def _accept_aggregate(self, lst) -> None:
        while True:
            try:
                sock, _ = lst.accept()
            except OSError:
                return
            conn = Conn(sock)
            state = {"cid": None}

            def on_msg(m, conn=conn, state=state):
                state["cid"] = self._handle(conn, m, state["cid"])
                if isinstance(m, Join):
                    with self._lock:
                        rec = self._consumers.get(state["cid"])
                        if rec is not None and rec.conn is conn:
                            return HANDOFF  # admitted: the hub reads this socket from now on
                return None

            def on_handoff(pending, conn=conn, state=state):
                with self._lock:
                    # the consumer may have been dropped (failed send, rejoin)
                    # between admission and this handoff: its fd is then closed
                    # or already reused, and must not be handed to the hub
                    rec = self._consumers.get(state["cid"])
                    if rec is None or rec.conn is not conn or conn.closed:
                        return
                    fd = conn.sock.fileno()
                    if fd < 0:
                        return
                    self._hub_fds[fd] = state["cid"]
                    self._hub.add(fd, state["cid"], pending)

            def on_close(conn=conn, state=state):
                with self._lock:
                    cid = state["cid"]
                    rec = self._consumers.get(cid)
                    if rec is not None and rec.conn is conn:
                        self._drop(cid, "disconnect")

            conn.start_reader(on_msg, on_close, "agg-reader", on_handoff)

    def _handle(self, conn: Conn, msg, cid):
        now = time.monotonic()
        if isinstance(msg, Ack):
            self._ack_q.append((msg, now))  # deque.append is atomic: no lock on the hot path
            return cid
        with self._lock:
            if isinstance(msg, Join):
                return self._handle_join(conn, msg, now)
            if isinstance(msg, Heartbeat):
                rec = self._consumers.get(msg.consumer_id)
                if rec is not None:
                    rec.last_heartbeat = now
            elif isinstance(msg, Bye):
                self._drain_acks()
                if msg.consumer_id in self._consumers:
                    self._drop(msg.consumer_id, "bye")
        return cid

    def _drain_hub(self) -> None:
        """Hub events: Acks join the ack queue; heartbeats, Byes and closed
        sockets are applied here (caller holds the lock)."""
        for kind, cid, epoch, bi, t, fd in self._hub.drain():
            if kind == 4:
                self._ack_q.append((Ack(cid, epoch, bi), t))
            elif kind == 5:
                rec = self._consumers.get(cid)
                if rec is not None:
                    rec.last_heartbeat = max(rec.last_heartbeat, t)
            elif kind == 8:
                self._drain_acks(hub=False)
                if cid in self._consumers:
                    self._drop(cid, "bye")
            else:  # connection closed / protocol error
                owner = self._hub_fds.pop(fd, None)
                rec = self._consumers.get(owner)
                if rec is not None and rec.conn is not None and rec.conn.sock.fileno() == fd:
                    self._drain_acks(hub=False)
                    self._drop(owner, "disconnect")

    def _drain_acks(self, hub: bool = True) -> None:
        """Fold queued wire Acks into the ledger (caller holds the lock)."""
        if hub:
            self._drain_hub()
        q = self._ack_q
        if not q:
            return
        L = max(1, len(self._loader))
        n, last = 0, None
        while q:
            try:
                msg, now = q.popleft()
            except IndexError:
                break
            last = now
            rec = self._consumers.get(msg.consumer_id)
            if rec is None or not rec.admitted:
                continue
            rec.last_heartbeat = max(rec.last_heartbeat, now)
            n += 1
            if rec.batch_size and rec.batch_size != self._per_slot:
                # heterogeneous consumer: its batch j fully covers the producer
                # batches before (j+1)*b // B; its last batch covers the epoch
                if rec.ack_epoch != msg.epoch:
                    rec.ack_epoch, rec.ack_k = msg.epoch, 0
                lc = rebatch_epoch_len(self._samples, L, self._per_slot, rec.batch_size)
                upto = L if msg.batch_index >= lc - 1 else min(
                    L, (msg.batch_index + 1) * rec.batch_size // self._per_slot)
                for k in range(rec.ack_k, upto):
                    self._ledger.ack(msg.consumer_id, seq_of(msg.epoch, k, L))
                rec.ack_k = max(rec.ack_k, upto)
                if upto:
                    rec.ack_seq = max(rec.ack_seq, seq_of(msg.epoch, upto - 1, L))
            else:
                seq = seq_of(msg.epoch, msg.batch_index, L)
                self._ledger.ack(msg.consumer_id, seq)
                rec.ack_seq = max(rec.ack_seq, seq)
        self.stats["acks"] += n
        if n:
            self._ledger.sample_drift(last, self._consumers.values())
            self._lock.notify_all()

    def _handle_join(self, conn: Conn, msg: Join, now: float):
        if msg.protocol_version not in SUPPORTED_VERSIONS or msg.consumer_id == MONITOR_ID:
            conn.close()
            return None
        # broadcast identification may lag the Join: wait briefly for it
        deadline = now + self._hb_timeout
        while msg.consumer_id not in self._bcast_pending and \
                not (msg.consumer_id in self._consumers and self._consumers[msg.consumer_id].bcast):
            if not self._lock.wait(timeout=max(0.0, deadline - time.monotonic())):
                conn.close()
                return None
        cid = msg.consumer_id
        bcast = self._bcast_pending.pop(cid, None)
        if cid in self._consumers:  # rejoin with the same id
            old = self._consumers[cid]
            bcast = bcast or old.bcast
            self._drop(cid, "rejoined", close_bcast=False)
        while self._ring is None:  # ring geometry comes from the first batch
            self._lock.wait(timeout=0.05)
            if self._closed:
                conn.close()
                return None
        dev = self.device if msg.device < 0 else msg.device
        bsz = msg.batch_size if msg.batch_size != self._per_slot else 0
        k = self._ring_for_device(dev)
        if k is None or (bsz and not self._rebatch_ok(bsz)):
            conn.close()  # no ring on that GPU / batch size not servable: no Welcome
            return None
        cursor = self._alloc_cursor(now)
        if cursor is None:
            conn.close()  # cursor table exhausted
            return None
        rec = ConsumerRecord(consumer_id=cid, cursor=cursor, last_heartbeat=now,
                             join_epoch=self._epoch, conn=conn, bcast=bcast, device=dev,
                             batch_size=bsz, ring=k)
        L = max(1, len(self._loader))
        progress = self._announced_in_epoch if self._epoch_started else 0
        code = admission_code(progress, L, self._fraction)
        q0 = seq_of(self._epoch, 0, L)
        if bsz and code == ADMIT_RUBBERBAND:
            code = ADMIT_WAIT  # replayed slots are producer batches; rebatching starts at an epoch
        if code in (ADMIT_IMMEDIATE, ADMIT_RUBBERBAND):
            rec.admitted = True
            self._rings[k].set_cursor(rec.cursor, q0 - 1)
            rec.ack_seq = q0 - 1  # ack cursor baseline (bs/producer.py:626-634)
            self._hub.set_acked(cid, q0 - 1)
            welcome = Welcome(cid, self._epoch, L, progress if code == ADMIT_RUBBERBAND else 0,
                              self._depth, code)
        else:
            rec.waiting_for_epoch = self._epoch + 1
            welcome = Welcome(cid, self._epoch + 1, L, 0, self._depth, ADMIT_WAIT)
        self._consumers[cid] = rec
        try:
            # ring descriptor first (private channel), then the Welcome
            conn.send(Announce(sg.RING_EPOCH, rec.cursor, self._descriptor_for(k).name(), 0,
                               DType.U8, (0,), 0))
            conn.send(welcome)
            if code == ADMIT_RUBBERBAND:
                for q in range(q0, q0 + progress):
                    anns = self._retained.get(q)
                    if anns is not None:
                        self._ledger.pending.setdefault(q, set()).add(cid)
                        conn.send(anns[k])
        except OSError:
            self._drop(cid, "disconnect")
        self._cver += 1
        self._lock.notify_all()
        return cid

    @property
    def cursor_quarantine_s(self) -> float:
        """How long a departed consumer's cursor word rests before reuse."""
        return 2 * self._hb_timeout

    def _alloc_cursor(self, now: float) -> int | None:
        """A cursor index valid in every ring (the cursor tables are parallel)."""
        if self._free_cursors and now - self._free_cursors[0][1] >= self.cursor_quarantine_s:
            return self._free_cursors.popleft()[0]
        if self._next_cursor < self._max_consumers:
            self._next_cursor += 1
            return self._next_cursor - 1
        return None

    def _drop(self, cid: int, reason: str, close_bcast: bool = True) -> None:
        rec = self._consumers.pop(cid, None)
        if rec is None:
            return
        now = time.monotonic()
        self.drops.append((cid, reason, now))
        self._hub.set_acked(cid, SENTINEL_MIN)  # no flow-gate wait on a departed consumer
        if rec.ring in self._rings:
            self._rings[rec.ring].evict(rec.cursor)  # unblocks every wait on this consumer
        if reason != "timeout":
            self._free_cursors.append((rec.cursor, now))
        self._ledger.remove_consumer(cid)
        if reason == "timeout":
            self.stats["evictions"] += 1
        if rec.conn is not None and not rec.conn.closed:
            fd = rec.conn.sock.fileno()
            if self._hub_fds.pop(fd, None) is not None:
                self._hub.remove(fd)  # stop reading before the fd can be reused
        for c in (rec.conn, rec.bcast if close_bcast else None):
            if c is not None:
                c.close()
        self._cver += 1
        self._lock.notify_all()

    def _sweep_loop(self) -> None:
        while not self._closed:
            time.sleep(self._poll)
            now = time.monotonic()
            with self._lock:
                self._drain_acks()
                for cid in [c for c, r in self._consumers.items()
                            if now - r.last_heartbeat > self._hb_timeout]:
                    self._drop(cid, "timeout")

    def _send_all(self, msg) -> None:
        data = encode(msg)
        for rec in list(self._consumers.values()):
            if rec.bcast is None:
                continue
            try:
                rec.bcast.send_raw(data)
            except OSError:
                self._drop(rec.consumer_id, "disconnect")
        for c in list(self._monitors):
            try:
                c.send_raw(data)
            except OSError:
                self._monitors.remove(c)
                self._cver += 1

    def _admitted(self):
        return [r for r in self._consumers.values() if r.admitted]

    # -- the epoch iterator -------------------------------------------------
    def __len__(self) -> int:
        return len(self._loader)

    def __iter__(self):
        if self._closed:
            raise ProducerClosed("join() was already called")
        self._start()
        L = len(self._loader)
        it = iter(self._loader) if not self._device_loader else None
        first = None
        if it is not None and L > 0:
            first = next(it)  # fixes the slot size before any consumer is admitted
            with self._lock:
                self._set_geometry(first)
                self._ensure_ring(self._pair_nbytes(first))
        with self._lock:
            need = 1 if self._barrier_met else self._min_consumers
            self._lock.wait_for(lambda: self._closed or len(self._admitted()) + sum(
                1 for r in self._consumers.values() if r.waiting_for_epoch == self._epoch) >= need)
            self._barrier_met = True
        for index in range(L):
            batch = None
            if it is not None:
                batch = first if index == 0 else next(it)
            if index == 0:
                self._start_epoch(L)
            self._publish(index, batch)
            yield None
        self._flush_pending()
        with self._lock:
            self._send_all(EpochEnd(self._epoch))
            self._drop_retention()
            self._epoch += 1
            self._announced_in_epoch = 0
            self._epoch_started = False

    @staticmethod
    def _pair_nbytes(batch) -> int:
        inp, tgt = batch
        n = 0
        for a in (inp, tgt):
            n += int(np.prod(getattr(a, "shape", ()))) * int(getattr(a, "itemsize", 0) or
                                                              a.element_size())
        return n

    def _start_epoch(self, L: int) -> None:
        with self._lock:
            q0 = seq_of(self._epoch, 0, L)
            for rec in self._consumers.values():
                if rec.waiting_for_epoch == self._epoch:
                    rec.waiting_for_epoch = None
                    rec.admitted = True
                    rec.ack_seq = q0 - 1
                    self._hub.set_acked(rec.consumer_id, q0 - 1)
                    if rec.ring in self._rings:
                        self._rings[rec.ring].set_cursor(rec.cursor, q0 - 1)
            self._epoch_started = True
            self._announced_in_epoch = 0
            self._retained.clear()
            self._cver += 1
            window = retention_window(self._fraction, L)
            if window > 0 and self._rings:
                for ring in self._rings.values():
                    ring.set_cursor(self._retention_cursor, q0 - 1)
                self._retention_active = True
            self._send_all(EpochStart(self._epoch, L))

    def _drop_retention(self) -> None:
        if self._retention_active:
            for ring in self._rings.values():
                ring.evict(self._retention_cursor)
            self._cver += 1
        self._retention_active = False

    # -- the one-GPU device-loader fast path ------------------------------------
    def _fast_ok(self) -> bool:
        return (self._device_loader and not self._multi and self._ring is not None and
                self._ring.host_control)

    def _fast_refresh(self) -> None:
        """Push the consumer lists to the native path (caller holds the lock)."""
        admitted = self._admitted()
        ack_ids = [r.consumer_id for r in admitted if not r.batch_size]
        live = [r.cursor for r in admitted]
        if self._retention_active:
            live.append(self._retention_cursor)
        fds, owner = [], {}
        for r in self._consumers.values():
            if r.bcast is not None and not r.bcast.closed:
                fd = r.bcast.sock.fileno()
                if fd >= 0:
                    fds.append(fd)
                    owner[fd] = r.consumer_id
        for c in self._monitors:
            fd = c.sock.fileno()
            if fd >= 0:
                fds.append(fd)
                owner[fd] = c
        self._facade.set_consumers(ack_ids, live, fds)
        self._facade_fds = owner
        self._fast_ids = [r.consumer_id for r in admitted]
        self._fast_live = live
        self._facade_ver = self._cver

    def _publish_fast(self, index: int) -> None:
        """_publish for one GPU and a CollateLoader-style device loader: the flow
        gate, the fused launch (+ CRC) and the Announce of each batch run in
        native code (hub.Facade); Python keeps the ledger and admission."""
        import torch

        from .hub import Facade

        ld, ring = self._loader, self._ring
        L = len(ld)
        q = seq_of(self._epoch, index, L)
        with self._lock:
            self._lock.wait_for(lambda: self._admitted() or self._closed)
            if self._closed:
                raise ProducerClosed("producer closed")
            if self._facade is None:
                self._facade = Facade()
            if self._facade_epoch != self._epoch:
                a = ld.produce_args(self._epoch, with_crc=self._crc if self._checksum else None)
                a.gate = GATE_HOST
                in_dt, in_shape = ld.input_dtype, tuple(ld.input_shape)
                tg_dt, tg_shape = ld.target_dtype, tuple(ld.target_shape)
                in_bytes, nbytes = ld.input_nbytes, ld.batch_nbytes
                self._hdr_reserved = sg.pack_pair_reserved(int(in_dt), len(in_shape), int(tg_dt),
                                                           len(tg_shape), in_bytes)
                self._hdr_key = (int(in_dt), in_shape, int(tg_dt), tg_shape, in_bytes, nbytes)
                self._fast_meta = (nbytes, (*in_shape, *tg_shape))
                header = sg.pack_header(self._epoch, 0, DType.U8, (nbytes,), nbytes, 0,
                                        reserved=self._hdr_reserved,
                                        extra_slots=(*in_shape, *tg_shape))
                self._facade.set_batch(self._hub, ring, a, self._stream, self._depth,
                                       self._ring_ids[0], header, nbytes,
                                       self._crc if self._checksum else None,
                                       self._crc_host if self._checksum else None,
                                       self._events)
                self._facade_epoch = self._epoch
            if self._facade_ver != self._cver:
                self._fast_refresh()
        if self._pending_ann is not None and self._pending_ann[0] <= q - self._depth:
            self._flush_pending()  # (buffer_depth 1: the gate waits for that batch's acks)
        while self._pend_fast and self._pend_fast[0][0] <= q - self._depth:
            self._announce_crc(self._pend_fast.popleft())  # the gate waits for its acks
        cur = (q, index, ring.slot_of(q), self._epoch)
        # announce in the same native call: this batch (no checksum), or the
        # one ANN_LAG launches back, whose CRC the kernel stored before publishing
        ann = None
        if not self._checksum:
            ann = cur
        elif len(self._pend_fast) >= ANN_LAG:
            ann = self._pend_fast[0]
        import contextlib

        here = torch.cuda.current_device() == self.device  # (the usual case: no switch)
        # with a checksum the launch and the Announce are two native calls: the
        # Python bookkeeping of the previous Announce runs between them, while
        # the GPU finishes the batch about to be announced
        split = self._checksum and ann is not None
        while True:
            with contextlib.nullcontext() if here else torch.cuda.device(self.device):
                res = self._facade.step(q, index, self._chain_ok, 0.1,
                                        None if ann is None or split else (ann[0], ann[3], ann[1]),
                                        self._checksum)
            if res is not None:
                break
            if self._closed:
                raise ProducerClosed("producer closed while waiting for consumers")
            with self._lock:  # evicted / departed consumers leave the gate
                if self._facade_ver != self._cver:
                    self._fast_refresh()
        # the native path knows whether its stream ends in a fused kernel (a
        # checksum read-back copy breaks the chain only for unfused geometries)
        self._chain_ok = True
        if split:
            self._settle_fast()
            with contextlib.nullcontext() if here else torch.cuda.device(self.device):
                res = self._facade.announce(ann[0], ann[3], ann[1], True)
        if ann is not None:  # live = announced and not yet released
            self._sample_live(ann[0], {0: self._fast_live})
        if self._checksum:
            if ann is not None:
                self._pend_fast.popleft()
            self._pend_fast.append(cur)
        if ann is not None:
            if split:
                self._settled = (ann, res)  # bookkept at the next launch (or a flush)
            else:
                self._announced_fast(ann, *res)

    def _settle_fast(self) -> None:
        """Bookkeeping of the last Announce the split fast path sent."""
        done, self._settled = self._settled, None
        if done is not None:
            self._announced_fast(done[0], *done[1])

    def _announce_fast(self, p, with_crc: bool) -> None:
        q, index, slot, epoch = p
        self._announced_fast(p, *self._facade.announce(q, epoch, index, with_crc))

    def _announced_fast(self, p, crc: int, failed) -> None:
        """Bookkeeping of an Announce the native path sent."""
        q, index, slot, epoch = p
        L = len(self._loader)
        with self._lock:
            for fd in failed:
                who = self._facade_fds.get(fd)
                if isinstance(who, int):
                    self._drop(who, "disconnect")
                elif who in self._monitors:
                    self._monitors.remove(who)
                    self._cver += 1
            self._ledger.add(q, self._fast_ids)
            self.batches.append((epoch, index, crc))
            self._announced_in_epoch = index + 1
            self.stats["announced"] += 1
            if self._retention_active:  # replayable announces for rubberband joiners
                nbytes, extra = self._fast_meta
                header = sg.pack_header(epoch, index, DType.U8, (nbytes,), nbytes, crc,
                                        reserved=self._hdr_reserved, extra_slots=extra)
                self._retained[q] = {0: Announce(epoch, index,
                                                 sg.slot_name(self._ring_ids[0], slot, header),
                                                 nbytes, DType.U8, (nbytes,), crc)}
                if self._announced_in_epoch >= retention_window(self._fraction, L):
                    self._drop_retention()
            self._since_drain += 1
            if self._since_drain >= 16:  # wire Acks fold into the ledger in bulk
                self._since_drain = 0
                self._drain_acks()

    def _publish(self, index: int, batch) -> None:
        import torch

        if self._fast_ok():
            return self._publish_fast(index)
        L = len(self._loader)
        q = seq_of(self._epoch, index, L)
        if self._device_loader:
            ld = self._loader
            in_dt, in_shape = ld.input_dtype, tuple(ld.input_shape)
            tg_dt, tg_shape = ld.target_dtype, tuple(ld.target_shape)
            in_bytes, nbytes = ld.input_nbytes, ld.batch_nbytes
        else:
            inp, tgt = batch
            inp = torch.as_tensor(inp)
            tgt = torch.as_tensor(tgt)
            in_dt, tg_dt = dtype_of(inp), dtype_of(tgt)
            in_shape, tg_shape = tuple(inp.shape), tuple(tgt.shape)
            in_bytes = inp.numel() * inp.element_size()
            nbytes = in_bytes + tgt.numel() * tgt.element_size()
        with self._lock:
            self._ensure_ring(nbytes)
            self._lock.wait_for(lambda: self._admitted() or self._closed)
            admitted = self._admitted()
            # the reference's flow gate (bs/producer.py:230-238, sl/producer.py:
            # 291-294): announce only while fewer than buffer_depth batches await
            # acks, counted on the wire Acks the native hub has received (so the
            # ledger's drift series obeys the same bound).  Consumers with their
            # own batch size and the rubberband retention cursor only gate slot
            # reuse (retained-but-acked batches do not count, :182-184)
            depth_ids = [r.consumer_id for r in admitted if not r.batch_size]
            live_by_ring = {k: [r.cursor for r in admitted if r.ring == k]
                            for k in range(len(self._devices))}
            if self._retention_active:
                for lv in live_by_ring.values():
                    lv.append(self._retention_cursor)
        ring, stream = self._ring, self._stream
        slot = ring.slot_of(q)
        host_gated = all(r.host_control for r in self._rings.values())
        if self._pending_ann is not None and self._pending_ann[0] <= q - self._depth:
            self._flush_pending()  # (buffer_depth 1: the gate waits for that batch's acks)
        self._ack_gate(q, depth_ids)
        if host_gated:
            # slot-reuse gate on the host-shared cursors: the producer's streams
            # never park on a device wait, so no stream of this process
            # (in-process consumers included) can be blocked behind one
            self._host_gate(q, live_by_ring)
            self._live_lists = live_by_ring  # sampled when a batch is announced
        if self._two_stage and not self._checksum:
            self._publish_two_stage(q, index)
        elif self._multi and self._device_loader and not self._checksum:
            self._publish_group(q, index)
        elif self._device_loader and host_gated and not self._multi:
            # fused collate + target + publish; with checksum=True the device
            # CRC-32 of the slot follows on the same stream (tsb_produce_range)
            a = self._loader.produce_args(self._epoch,
                                          with_crc=self._crc if self._checksum else None)
            a.gate = GATE_HOST
            a.chain = int(self._chain_ok)  # the stream's previous op was our fused kernel
            with torch.cuda.device(self.device):
                produce_range(ring, a, q, index, 1, [], stream=stream)
                if self._checksum:
                    with torch.cuda.stream(stream):
                        self._crc_host[slot:slot + 1].copy_(self._crc[slot:slot + 1],
                                                            non_blocking=True)
                    self._events[slot].record(stream)
            self._chain_ok = not self._checksum
        else:
            if not host_gated and q > ring.slots:
                # bound host run-ahead: batch q-S (same slot) must have been published
                self._events[slot].synchronize()
            self._chain_ok = False
            for k, d in enumerate(self._devices):
                r, st = self._rings[k], self._streams[k]
                with torch.cuda.device(d), torch.cuda.stream(st):
                    if not host_gated:
                        r.wait_free(live_by_ring[k], q - r.slots, st)
                    base = r.slot_ptr(slot)
                    if self._device_loader:
                        self._loader.produce_into(base, self._epoch, index, st)
                    else:
                        view = r.view(slot, (nbytes,), torch.uint8)
                        view[:in_bytes].copy_(inp.contiguous().reshape(-1).view(torch.uint8),
                                              non_blocking=True)
                        view[in_bytes:nbytes].copy_(
                            tgt.contiguous().reshape(-1).view(torch.uint8), non_blocking=True)
                    if self._checksum and k == 0:
                        dp.crc32(base, nbytes, self._crc[slot:slot + 1], st)
                        self._crc_host[slot:slot + 1].copy_(self._crc[slot:slot + 1],
                                                            non_blocking=True)
                    r.publish(slot, q, st)
                    if k == 0:
                        self._events[slot].record(st)
        hkey = (int(in_dt), in_shape, int(tg_dt), tg_shape, in_bytes, nbytes)
        if self._hdr_key != hkey:  # the pair layout is fixed for a loader: pack it once
            self._hdr_key = hkey
            self._hdr_reserved = sg.pack_pair_reserved(int(in_dt), len(in_shape), int(tg_dt),
                                                       len(tg_shape), in_bytes)
        cur = (q, index, slot, nbytes, (*in_shape, *tg_shape), self._epoch)
        if not self._checksum:
            self._announce(cur, 0)
            return
        prev, self._pending_ann = self._pending_ann, cur
        if prev is not None:
            self._announce_crc(prev)

    def _announce_crc(self, p) -> None:
        """Announce a batch whose device CRC-32 was enqueued (waits for it)."""
        self._settle_fast()  # announces are bookkept in order
        if len(p) == 4:  # enqueued by the native fast path
            self._announce_fast(p, True)
            return
        slot = p[2]
        self._events[slot].synchronize()
        self._announce(p, int(self._crc_host[slot]) & 0xFFFFFFFF)

    def _flush_pending(self) -> None:
        self._settle_fast()
        p, self._pending_ann = self._pending_ann, None
        if p is not None:
            self._announce_crc(p)
        while self._pend_fast:
            self._announce_crc(self._pend_fast.popleft())

    def _announce(self, p, crc: int) -> None:
        """Announce (q, index, slot, nbytes, extra shape slots, epoch) with its
        checksum to every consumer: the 80-byte segment header rides in the
        slot name (bs/producer.py:506-534)."""
        q, index, slot, nbytes, extra, epoch = p
        header = sg.pack_header(epoch, index, DType.U8, (nbytes,), nbytes, crc,
                                reserved=self._hdr_reserved, extra_slots=extra)
        anns = {k: Announce(epoch, index, sg.slot_name(self._ring_ids[k], slot, header),
                            nbytes, DType.U8, (nbytes,), crc) for k in self._rings}
        L = len(self._loader)
        with self._lock:
            self._drain_acks()
            self._ledger.add(q, [r.consumer_id for r in self._admitted()])
            self._send_announces(anns)
            self.batches.append((epoch, index, crc))
            self._announced_in_epoch = index + 1
            self.stats["announced"] += 1
            if self._live_lists is not None:  # live = announced, not released
                self._sample_live(q, self._live_lists)
            window = retention_window(self._fraction, L)
            if self._retention_active:
                self._retained[q] = anns
                if self._announced_in_epoch >= window:
                    self._drop_retention()

    def _order_on(self, dev: int, epoch: int):
        """The epoch order resident on `dev` (a shard's kernel reads its indices locally)."""
        import torch

        key = (dev, epoch)
        if key not in self._orders:
            for k in [k for k in self._orders if k[1] != epoch]:
                del self._orders[k]
            host, _ = self._loader.order(epoch)
            self._orders[key] = torch.from_numpy(host).to(f"cuda:{dev}")
        return self._orders[key]

    def _ack_gate(self, q: int, ids) -> None:
        """The reference's flow gate (bs/producer.py:230-238): batch q is
        announced only once every consumer acked q - buffer_depth on the wire,
        i.e. fewer than buffer_depth announced batches await acks.  The native
        hub counts the Acks as it decodes them (no interpreter on the wait)."""
        need = q - self._depth
        while not self._hub.wait_acked(ids, need, timeout_s=0.1):
            if self._closed:
                raise ProducerClosed("producer closed while waiting for consumers")
            with self._lock:  # evicted / departed consumers leave the gate
                ids = [i for i in ids if i in self._consumers]

    def _host_gate(self, q: int, live_by_ring) -> None:
        """Block until every live cursor of every ring released batch q-S
        (slot reuse)."""
        need = q - self._ring.slots
        if need <= 0:
            return
        for k, ring in self._rings.items():
            live = live_by_ring[k]
            if ring.released(live, need):  # the common case: no wait, no native call
                continue
            while not ring.host_gate(live, need, timeout_s=0.1):
                if self._closed:
                    raise ProducerClosed("producer closed while waiting for consumers")

    def _sample_live(self, q: int, live_by_ring) -> None:
        """Live slots when batch q is published: batches announced but not yet
        released by every live cursor (SPEC.md:528 memory bound: <= N+1 outside
        the rubberband window)."""
        low = None
        for k, ring in self._rings.items():
            cur = ring.cursor_words
            for c in live_by_ring[k]:
                v = int(cur[c])
                if v < SENTINEL_MIN and (low is None or v < low):
                    low = v
        if low is None:
            return
        live = q - low
        key = "live_max_window" if self._retention_active else "live_max"
        if live > self.stats[key]:
            self.stats[key] = live

    def _publish_group(self, q: int, index: int) -> None:
        """Multi-GPU: every device produces its shard of the batch straight into
        the slot of every device's ring (sharded), or the first device produces
        the whole batch into every ring (star); publish is fused into the kernel
        and the flow gate runs on the host (tsb_produce_group)."""
        import torch

        G = len(self._devices)
        writers = list(range(G)) if self._sharded else [0]
        key = (self._epoch, tuple(writers))
        if getattr(self, "_group_cache", (None,))[0] != key:
            from ._lib import ProduceArgs

            base = self._loader.produce_args(self._epoch)
            args = []
            for k in writers:
                a = ProduceArgs.from_buffer_copy(base)
                o = self._order_on(self._devices[k], self._epoch)
                a.d_order = o.data_ptr()
                a._keep = (o,)
                a.gate = GATE_HOST
                args.append(a)
            self._group_cache = (key, args)
        args = self._group_cache[1]
        for a in args:
            a.chain = int(self._chain_ok)  # each writer's stream: previous op was its kernel
        produce_group_multi([self._rings[k] for k in range(G)], args, writers,
                            [self._devices[k] for k in writers],
                            [self._streams[k] for k in writers], q, index, 1,
                            [[] for _ in range(G)])  # gated on the host already (_host_gate)
        self._chain_ok = True

    def _publish_two_stage(self, q: int, index: int) -> None:
        """Multi-GPU, two-stage: stage 1 -- every device gathers its 1/G rows of
        batch q (u8 + target indices) into slot q of every device's input ring
        (tsb_produce_group_multi, gated on the input rings' single cursor);
        stage 2 -- each device collates the whole staged batch into its own
        ring on a second stream (tsb_restage_collate: the kernel publishes the
        output slot and releases the input slot).  The output rings were gated
        on the host already (_host_gate)."""
        from ._lib import ProduceArgs

        G = len(self._devices)
        key = (self._epoch, "inputs")
        if getattr(self, "_group_cache", (None,))[0] != key:
            gbase = self._gather_loader.produce_args(self._epoch)
            abase = self._loader.produce_args(self._epoch)
            gargs, aargs = [], []
            for k in range(G):
                a = ProduceArgs.from_buffer_copy(gbase)
                o = self._order_on(self._devices[k], self._epoch)
                a.d_order = o.data_ptr()
                a._keep = (o,)
                a.gate = GATE_HOST
                gargs.append(a)
                a2 = ProduceArgs.from_buffer_copy(abase)
                a2._keep = getattr(abase, "_keep", None)
                a2.ingest = self._tables[k].handle
                a2.gate = GATE_HOST
                aargs.append(a2)
            self._group_cache = (key, (gargs, aargs))
        gargs, aargs = self._group_cache[1]
        for a in gargs:
            a.chain = int(self._chain_ok)
        produce_group_multi([self._in_rings[k] for k in range(G)], gargs, list(range(G)),
                            self._devices, [self._streams[k] for k in range(G)], q, index, 1,
                            [[0] for _ in range(G)])
        self._chain_ok = True
        import torch

        for k, d in enumerate(self._devices):
            aargs[k].chain = int(self._chain2_ok)
            with torch.cuda.device(d):
                restage_collate(self._in_rings[k], 0, self._rings[k], aargs[k], q, 1, [],
                                stream=self._streams2[k])
        self._chain2_ok = True

    def _send_announces(self, anns: dict) -> None:
        """Announce a batch: each consumer gets the slot name of its own GPU's ring."""
        data = {d: encode(a) for d, a in anns.items()}
        by_ring: dict[int, list] = {}
        for rec in self._consumers.values():
            if rec.bcast is not None and not rec.bcast.closed:
                by_ring.setdefault(rec.ring, []).append(rec)
        for k, recs in by_ring.items():  # one native call per ring: no per-consumer Python
            failed = set(Hub.broadcast([r.bcast.sock.fileno() for r in recs], data[k]))
            for r in recs:
                if r.bcast.sock.fileno() in failed:
                    self._drop(r.consumer_id, "disconnect")
        for c in list(self._monitors):
            try:
                c.send_raw(data[0])
            except OSError:
                self._monitors.remove(c)
                self._cver += 1

    # -- shutdown ---------------------------------------------------------------
    def join(self, drain_timeout_s: float = 10.0) -> None:
        """Wait for outstanding acks, broadcast Shutdown, release the ring."""
        if self._closed:
            return
        self._flush_pending()
        deadline = time.monotonic() + drain_timeout_s
        with self._lock:
            while time.monotonic() < deadline:
                self._drain_acks()
                if not self._ledger.pending:
                    break
                self._lock.wait(0.002)
            self._drain_acks()
            self._send_all(Shutdown())
        # device drain: every live consumer released the last batch (bounded wait)
        if self._ring is not None:
            with self._lock:
                cursors = [(self._rings[r.ring], r.cursor) for r in self._admitted()]
            final = seq_of(self._epoch, 0, max(1, len(self._loader))) - 1
            while cursors and time.monotonic() < deadline:
                if all(ring.read_cursor(c) >= final for ring, c in cursors):
                    break
                time.sleep(0.005)
        with self._lock:
            self._closed = True
            for lst in self._listeners:
                try:
                    lst.close()
                except OSError:
                    pass
            for cid in list(self._consumers):
                self._drop(cid, "shutdown")
            for c in self._monitors:
                c.close()
            self._lock.notify_all()

    @property
    def drift_max(self) -> int:
        """Largest wire-ack spread between admitted consumers seen so far
        (SPEC.md:524): the hub samples it at every Ack, the ledger at every drain."""
        return max(self._ledger.drift_max, self._hub.drift_max())

    def close(self) -> None:
        """Release the device ring (after join()).  Consumers must be gone."""
        self.join(0.0)
        for st in list(self._streams.values()) + list(self._streams2.values()):
            st.synchronize()
        with self._lock:  # the sweeper drains the hub under the same lock
            self._hub.close()
            if self._facade is not None:
                self._facade.close()
                self._facade = None
        for d, ring in self._rings.items():
            _RINGS.pop(self._ring_ids[d], None)
            ring.close()
        self._rings.clear()
        for ring in self._in_rings.values():
            ring.close()
        self._in_rings.clear()
        self._tables.clear()
        self._ring = None

    def __del__(self):
        try:
            if self._ring is not None and not self._closed:
                self.join(0.0)
        except Exception:
            pass


__all__ = ["TensorProducer", "ProducerClosed"]
