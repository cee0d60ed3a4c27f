"""Native control-plane hub (csrc/tsb_hub.cpp): per-batch socket work of the
producer -- decoding every consumer's wire Acks and writing every Announce --
off the interpreter lock.  The handshake stays in Python (transport.Conn);
an admitted consumer's aggregate socket is handed to the hub."""

from __future__ import annotations

import ctypes

from . import _lib
from .wire import Ack, Bye, Heartbeat

KIND_CLOSED = 0
_KINDS = {4: Ack, 5: Heartbeat, 8: Bye}


class Hub:
    def __init__(self, cap: int = 4096):
        h = ctypes.c_void_p()
        _lib.call("tsb_hub_create", ctypes.byref(h))
        self._h = h.value
        self._buf = (_lib.HubEvent * cap)()
        self._cap = cap
        self._n = ctypes.c_int(0)
        self._L = _lib.load()

    def add(self, fd: int, consumer_id: int, pending: bytes = b"") -> None:
        buf = ctypes.create_string_buffer(pending, len(pending)) if pending else None
        _lib.call("tsb_hub_add", self._h, fd, consumer_id, buf, len(pending))

    def remove(self, fd: int) -> None:
        if self._h:  # (closed hub: nothing is read anymore)
            _lib.call("tsb_hub_remove", self._h, fd)

    def drain(self):
        """[(kind, consumer_id, epoch, batch_index, t_monotonic_s, fd)] received so far;
        kind is the wire kind (4 Ack, 5 Heartbeat, 8 Bye) or 0 = connection closed."""
        out = []
        while self._h:
            _lib.check(self._L.tsb_hub_drain(self._h, self._buf, self._cap,
                                             ctypes.byref(self._n)), "tsb_hub_drain")
            n = self._n.value
            b = self._buf
            out.extend((b[i].kind, b[i].consumer_id, b[i].epoch, b[i].batch_index,
                        b[i].t_us * 1e-6, b[i].fd) for i in range(n))
            if n < self._cap:
                return out
        return out

    # -- the reference's flow gate on received wire Acks (bs/producer.py:230-238)
    def set_epoch_len(self, epoch_len: int) -> None:
        _lib.call("tsb_hub_set_epoch_len", self._h, epoch_len)

    def set_acked(self, consumer_id: int, seq: int) -> None:
        """Assign a consumer's acked seq (admission baseline; a sentinel on drop)."""
        if self._h:
            _lib.call("tsb_hub_set_acked", self._h, consumer_id, seq)

    def read_acked(self, consumer_id: int) -> int:
        v = ctypes.c_uint64()
        _lib.call("tsb_hub_read_acked", self._h, consumer_id, ctypes.byref(v))
        return v.value

    def wait_acked(self, consumer_ids, need: int, timeout_s: float = -1.0) -> bool:
        """Block until every listed consumer acked seq >= need; False on timeout."""
        ids = list(consumer_ids)
        if not ids or need <= 0:
            return True
        arr = (ctypes.c_uint64 * len(ids))(*ids)
        rc = self._L.tsb_hub_wait_acked(self._h, arr, len(ids), need,
                                        -1 if timeout_s < 0 else int(timeout_s * 1e6))
        if rc == _lib.TSB_ERR_STALE:
            return False
        _lib.check(rc, "tsb_hub_wait_acked")
        return True

    def drift_max(self) -> int:
        """Largest acked-seq spread over registered consumers seen at any Ack."""
        if not self._h:
            return 0
        v = ctypes.c_uint64()
        _lib.call("tsb_hub_drift_max", self._h, ctypes.byref(v))
        return v.value

    @staticmethod
    def broadcast(fds, frame: bytes) -> list:
        """Send `frame` to every fd; returns the fds whose send failed."""
        n = len(fds)
        if not n:
            return []
        arr = (ctypes.c_int * n)(*fds)
        failed = (ctypes.c_int * n)()
        _lib.call("tsb_hub_broadcast", arr, n, frame, len(frame), failed)
        return [fds[i] for i in range(n) if failed[i]]

    def close(self) -> None:
        h, self._h = self._h, None
        if h:
            self._L.tsb_hub_destroy(h)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Facade:
    """tsb_facade: the per-batch producer path (flow gate, fused launch,
    checksum read-back, Announce encode + broadcast) in two native calls."""

    def __init__(self):
        h = ctypes.c_void_p()
        _lib.call("tsb_facade_create", ctypes.byref(h))
        self._h = h.value
        self._L = _lib.load()
        self._keep = []
        self._failed = (ctypes.c_int * 1)()
        self._crc = ctypes.c_uint32(0)
        self.fds: list = []

    def set_batch(self, hub: Hub, ring, args, stream, depth: int, ring_id: int, header: bytes,
                  nbytes: int, d_crc=None, h_crc=None, events=None) -> None:
        from .ring import hold_for_stream

        evs = None
        if d_crc is not None:
            evs = (ctypes.c_void_p * ring.slots)(*[int(e.cuda_event) for e in events])
        hold_for_stream(args, stream)
        self._keep = [args, evs, header]
        _lib.call("tsb_facade_set_batch", self._h, hub._h, ring._h, ctypes.byref(args),
                  _lib.stream_handle(stream), depth, ring_id, header, nbytes,
                  None if d_crc is None else d_crc.data_ptr(),
                  None if h_crc is None else h_crc.data_ptr(), evs, ring.slots)

    def set_consumers(self, ack_ids, live, fds) -> None:
        n1, n2, n3 = len(ack_ids), len(live), len(fds)
        a = (ctypes.c_uint64 * max(1, n1))(*ack_ids)
        b = (ctypes.c_int * max(1, n2))(*live)
        c = (ctypes.c_int * max(1, n3))(*fds)
        self._failed = (ctypes.c_int * max(1, n3))()
        self.fds = list(fds)
        _lib.call("tsb_facade_set_consumers", self._h, a, n1, b, n2, c, n3)

    def produce(self, seq: int, index: int, chain: bool, timeout_s: float) -> bool:
        """False when the flow gate timed out (the caller re-checks shutdown)."""
        rc = self._L.tsb_facade_produce(self._h, seq, index, int(chain), int(timeout_s * 1e6))
        if rc == _lib.TSB_ERR_STALE:
            return False
        _lib.check(rc, "tsb_facade_produce")
        return True

    def step(self, seq: int, index: int, chain: bool, timeout_s: float, ann=None,
             with_crc: bool = False):
        """produce(seq) + announce(ann = (seq, epoch, index)) in one call:
        None when the flow gate timed out (nothing was produced), else
        (crc, failed fds) of the announce (or (0, []) with no announce)."""
        aq, ae, ai = ann if ann is not None else (0, 0, 0)
        rc = self._L.tsb_facade_step(self._h, seq, index, int(chain), int(timeout_s * 1e6), aq, ae,
                                     ai, int(with_crc), ctypes.byref(self._crc), self._failed)
        if rc == _lib.TSB_ERR_STALE:
            return None
        _lib.check(rc, "tsb_facade_step")
        if ann is None:
            return 0, []
        failed = [fd for i, fd in enumerate(self.fds) if self._failed[i]] if self.fds else []
        return self._crc.value, failed

    def announce(self, seq: int, epoch: int, index: int, with_crc: bool):
        """-> (crc, [fds whose send failed])."""
        _lib.check(self._L.tsb_facade_announce(self._h, seq, epoch, index, int(with_crc),
                                               ctypes.byref(self._crc), self._failed),
                   "tsb_facade_announce")
        failed = [fd for i, fd in enumerate(self.fds) if self._failed[i]] if self.fds else []
        return self._crc.value, failed

    def close(self) -> None:
        h, self._h = self._h, None
        if h:
            self._L.tsb_facade_destroy(h)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
