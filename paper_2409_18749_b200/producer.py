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
* release is device-counted: consumers advance a cursor word from their own
  CUDA stream; the producer's stream waits on the cursors before reusing a
  slot -- no host round trip on the data path;
* the reference's wire protocol is kept byte-for-byte (Join/Welcome/Announce/
  Ack/Heartbeat/EpochStart/EpochEnd/Bye/Shutdown); the Announce's segment
  name carries the slot and its 80-byte segment header (segment.py).

Keyword-only extensions: ``ring_slots`` (device ring depth; bounds drift),
``control`` ("host": ring control words in a host-shared, device-mapped
shm block -- evictions and map-and-ack consumers never touch a GPU channel;
"device": words in HBM), ``min_consumers`` (start barrier, bs/producer.py:73-76 -- the facade's
missing barrier is the start race noted in SURVEY.md §4), ``checksum``
(device CRC-32 of every batch into Announce.checksum), ``rubberband_fraction``
(late-join replay window, bs/producer.py:119-135; 0 = facade behaviour),
``device``.
"""

from __future__ import annotations

import os
import threading
import time

import numpy as np

from . import dataplane as dp
from . import segment as sg
from .errors import ProducerClosed
from .ledger import ConsumerRecord, Ledger, admission_code, retention_window, seq_of
from .ring import DeviceRing
from .transport import Conn, endpoints_from_env, listen
from .wire import (ADMIT_IMMEDIATE, ADMIT_RUBBERBAND, ADMIT_WAIT, PROTOCOL_VERSION, Ack, Announce,
                   Bye, DType, EpochEnd, EpochStart, Heartbeat, Join, Shutdown, Welcome, dtype_of,
                   encode)

MONITOR_ID = 0  # bs/producer.py:52-54: passive broadcast observers
_RINGS: dict[int, DeviceRing] = {}  # ring_id -> ring, for same-process consumers


def local_ring(ring_id: int):
    return _RINGS.get(ring_id)


class TensorProducer:
    def __init__(self, data_loader, broadcast: str | None = None, aggregate: str | None = None,
                 buffer_depth: int = 2, heartbeat_timeout_s: float = 5.0,
                 pause_poll_s: float = 0.05, *, ring_slots: int | None = None,
                 min_consumers: int = 1, checksum: bool = False,
                 rubberband_fraction: float = 0.0, max_consumers: int = 64,
                 device: int | None = None, control: str = "host"):
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
        self._checksum = checksum
        self._fraction = rubberband_fraction
        self._max_consumers = max_consumers
        self._ring_slots = ring_slots
        self._control = control
        self.device = torch.cuda.current_device() if device is None else device
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
        self._closed = False
        self._started = False
        self._listeners = []
        self._threads: list[threading.Thread] = []
        self._ring: DeviceRing | None = None
        self._stream = None
        self._events = []
        self._retained: dict[int, Announce] = {}  # seq -> announce (rubberband prefix)
        self._retention_active = False
        self.ring_id = (os.getpid() << 20) ^ (id(self) & 0xFFFFF)
        self.stats = {"announced": 0, "acks": 0, "evictions": 0}

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
        with torch.cuda.device(self.device):
            window = retention_window(self._fraction, max(1, len(self._loader)))
            slots = self._ring_slots or max(self._depth + 2 + window, 4)
            if slots <= window:
                raise ValueError(f"ring_slots={slots} must exceed the rubberband window {window}")
            # cursor index max_consumers is the producer's retention cursor
            self._ring = DeviceRing(slots, nbytes, self._max_consumers + 1, device=self.device,
                                    control=self._control)
            self._stream = torch.cuda.Stream(device=self.device)
            self._events = [torch.cuda.Event() for _ in range(slots)]
            self._crc = torch.zeros(slots, dtype=torch.int32, device=f"cuda:{self.device}")
            self._crc_host = torch.zeros(slots, dtype=torch.int32).pin_memory()
            _RINGS[self.ring_id] = self._ring
            self._descriptor = sg.RingDescriptor(
                self.ring_id, os.getpid(), self.device, slots, nbytes, self._max_consumers + 1,
                self._ring.export(), self._ring.control_name)
        self._lock.notify_all()

    @property
    def ring(self) -> DeviceRing | None:
        return self._ring

    @property
    def _retention_cursor(self) -> int:
        return self._max_consumers

    # -- server plumbing --------------------------------------------------
    def _start(self) -> None:
        if self._started:
            return
        self._started = True
        hint = self._batch_nbytes_hint()
        if hint is not None:
            with self._lock:
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
                        self._lock.notify_all()

            def on_close(conn=conn, state=state):
                with self._lock:
                    cid = state["cid"]
                    if cid == MONITOR_ID and conn in self._monitors:
                        self._monitors.remove(conn)
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

            def on_close(conn=conn, state=state):
                with self._lock:
                    cid = state["cid"]
                    rec = self._consumers.get(cid)
                    if rec is not None and rec.conn is conn:
                        self._drop(cid, "disconnect")

            conn.start_reader(on_msg, on_close, "agg-reader")

    def _handle(self, conn: Conn, msg, cid):
        now = time.monotonic()
        with self._lock:
            if isinstance(msg, Join):
                return self._handle_join(conn, msg, now)
            if isinstance(msg, Ack):
                rec = self._consumers.get(msg.consumer_id)
                if rec is None or not rec.admitted:
                    return cid
                rec.last_heartbeat = now
                L = max(1, len(self._loader))
                seq = seq_of(msg.epoch, msg.batch_index, L)
                self._ledger.ack(msg.consumer_id, seq)
                rec.ack_seq = max(rec.ack_seq, seq)
                self.stats["acks"] += 1
                self._ledger.sample_drift(now, self._consumers.values())
                self._lock.notify_all()
            elif isinstance(msg, Heartbeat):
                rec = self._consumers.get(msg.consumer_id)
                if rec is not None:
                    rec.last_heartbeat = now
            elif isinstance(msg, Bye):
                if msg.consumer_id in self._consumers:
                    self._drop(msg.consumer_id, "bye")
        return cid

    def _handle_join(self, conn: Conn, msg: Join, now: float):
        if msg.protocol_version != PROTOCOL_VERSION or msg.consumer_id == MONITOR_ID:
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
        if self._next_cursor >= self._max_consumers:
            conn.close()  # cursor table exhausted
            return None
        rec = ConsumerRecord(consumer_id=cid, cursor=self._next_cursor, last_heartbeat=now,
                             join_epoch=self._epoch, conn=conn, bcast=bcast)
        self._next_cursor += 1
        L = max(1, len(self._loader))
        progress = self._announced_in_epoch if self._epoch_started else 0
        code = admission_code(progress, L, self._fraction)
        q0 = seq_of(self._epoch, 0, L)
        if code in (ADMIT_IMMEDIATE, ADMIT_RUBBERBAND):
            rec.admitted = True
            self._ring.set_cursor(rec.cursor, q0 - 1)
            welcome = Welcome(cid, self._epoch, L, progress if code == ADMIT_RUBBERBAND else 0,
                              self._depth, code)
        else:
            rec.waiting_for_epoch = self._epoch + 1
            welcome = Welcome(cid, self._epoch + 1, L, 0, self._depth, ADMIT_WAIT)
        self._consumers[cid] = rec
        try:
            # ring descriptor first (private channel), then the Welcome
            conn.send(Announce(sg.RING_EPOCH, rec.cursor, self._descriptor.name(), 0, DType.U8,
                               (0,), 0))
            conn.send(welcome)
            if code == ADMIT_RUBBERBAND:
                for q in range(q0, q0 + progress):
                    ann = self._retained.get(q)
                    if ann is not None:
                        self._ledger.pending.setdefault(q, set()).add(cid)
                        conn.send(ann)
        except OSError:
            self._drop(cid, "disconnect")
        self._lock.notify_all()
        return cid

    def _drop(self, cid: int, reason: str, close_bcast: bool = True) -> None:
        rec = self._consumers.pop(cid, None)
        if rec is None:
            return
        if self._ring is not None:
            self._ring.evict(rec.cursor)  # unblocks every device wait on this consumer
        self._ledger.remove_consumer(cid)
        if reason == "timeout":
            self.stats["evictions"] += 1
        for c in (rec.conn, rec.bcast if close_bcast else None):
            if c is not None:
                c.close()
        self._lock.notify_all()

    def _sweep_loop(self) -> None:
        while not self._closed:
            time.sleep(self._poll)
            now = time.monotonic()
            with self._lock:
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
                    if self._ring is not None:
                        self._ring.set_cursor(rec.cursor, q0 - 1)
            self._epoch_started = True
            self._announced_in_epoch = 0
            self._retained.clear()
            window = retention_window(self._fraction, L)
            if window > 0 and self._ring is not None:
                self._ring.set_cursor(self._retention_cursor, q0 - 1)
                self._retention_active = True
            self._send_all(EpochStart(self._epoch, L))

    def _drop_retention(self) -> None:
        if self._retention_active and self._ring is not None:
            self._ring.evict(self._retention_cursor)
        self._retention_active = False

    def _publish(self, index: int, batch) -> None:
        import torch

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
            live = [r.cursor for r in self._admitted()]
            if self._retention_active:
                live.append(self._retention_cursor)
        ring, stream = self._ring, self._stream
        slot = ring.slot_of(q)
        # bound host run-ahead: batch q-S (same slot) must have been published
        if q > ring.slots:
            self._events[slot].synchronize()
        with torch.cuda.device(self.device), torch.cuda.stream(stream):
            ring.wait_free(live, q - ring.slots, stream)
            base = ring.slot_ptr(slot)
            if self._device_loader:
                self._loader.produce_into(base, self._epoch, index, stream)
            else:
                view = ring.view(slot, (nbytes,), torch.uint8)
                view[:in_bytes].copy_(inp.contiguous().reshape(-1).view(torch.uint8),
                                      non_blocking=True)
                view[in_bytes:nbytes].copy_(tgt.contiguous().reshape(-1).view(torch.uint8),
                                            non_blocking=True)
            if self._checksum:
                dp.crc32(base, nbytes, self._crc[slot:slot + 1], stream)
                self._crc_host[slot:slot + 1].copy_(self._crc[slot:slot + 1], non_blocking=True)
            ring.publish(slot, q, stream)
            self._events[slot].record(stream)
        crc = 0
        if self._checksum:
            self._events[slot].synchronize()
            crc = int(self._crc_host[slot]) & 0xFFFFFFFF
        reserved = sg.pack_pair_reserved(int(in_dt), len(in_shape), int(tg_dt), len(tg_shape),
                                         in_bytes)
        header = sg.pack_header(self._epoch, index, DType.U8, (nbytes,), nbytes, crc,
                                reserved=reserved, extra_slots=(*in_shape, *tg_shape))
        ann = Announce(self._epoch, index, sg.slot_name(self.ring_id, slot, header), nbytes,
                       DType.U8, (nbytes,), crc)
        with self._lock:
            self._ledger.add(q, [r.consumer_id for r in self._admitted()])
            self._send_all(ann)
            self._announced_in_epoch = index + 1
            self.stats["announced"] += 1
            window = retention_window(self._fraction, L)
            if self._retention_active:
                self._retained[q] = ann
                if self._announced_in_epoch >= window:
                    self._drop_retention()

    # -- shutdown ---------------------------------------------------------------
    def join(self, drain_timeout_s: float = 10.0) -> None:
        """Wait for outstanding acks, broadcast Shutdown, release the ring."""
        if self._closed:
            return
        deadline = time.monotonic() + drain_timeout_s
        with self._lock:
            self._lock.wait_for(lambda: not self._ledger.pending, timeout=drain_timeout_s)
            self._send_all(Shutdown())
        # device drain: every live consumer released the last batch (bounded wait)
        if self._ring is not None:
            with self._lock:
                cursors = [r.cursor for r in self._admitted()]
            final = seq_of(self._epoch, 0, max(1, len(self._loader))) - 1
            while cursors and time.monotonic() < deadline:
                if all(self._ring.read_cursor(c) >= final for c in cursors):
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

    def close(self) -> None:
        """Release the device ring (after join()).  Consumers must be gone."""
        self.join(0.0)
        if self._stream is not None:
            self._stream.synchronize()
        if self._ring is not None:
            _RINGS.pop(self.ring_id, None)
            self._ring.close()
            self._ring = None

    def __del__(self):
        try:
            if self._ring is not None and not self._closed:
                self.join(0.0)
        except Exception:
            pass


__all__ = ["TensorProducer", "ProducerClosed"]
