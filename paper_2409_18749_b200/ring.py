"""DeviceRing: the HBM batch ring that replaces the reference's per-batch
POSIX shm segments (payload.py:165-370) and its ack-gated release
(producer.py:169-252).

A ring is one device allocation holding ``slots`` payload slots plus a
control block of device words:

* ``ready[slot]``   -- global sequence number (1-based) of the batch the slot
  currently holds, written by the producer's stream after the batch is
  complete (release semantics);
* ``cursor[k]``     -- highest sequence consumer k has *released*; written by
  the consumer's stream once its work on that batch is done.

Batch with sequence q (q = epoch*epoch_len + index + 1) lives in slot
(q-1) % slots.  The producer may overwrite a slot for q only once every live
consumer released q - slots (device wait on the cursors), so a ring of S
slots bounds drift to S batches with no host round trip on the data path.
Eviction writes cursor = 2**62 (TSB_CURSOR_EVICTED) so no device wait can wedge
(producer.py:255-269).

Zero-copy views: same process -> the pointer; other processes on the same
GPU -> CUDA-IPC import of the whole allocation (handle shipped once, inside
the Announce's segment name).
"""

from __future__ import annotations

import ctypes
import mmap
import os

from . import _lib
from ._lib import IPC_HANDLE_BYTES, call, load

SENTINEL = 1 << 62  # TSB_CURSOR_EVICTED: positive under the memop wrap-around GEQ

_TORCH_TYPESTR = {
    "uint8": "|u1", "int8": "|i1", "int16": "<i2", "int32": "<i4", "int64": "<i8",
    "float32": "<f4", "float64": "<f8", "float16": "<f2", "bfloat16": "<i2",
}


class _CAI:
    """__cuda_array_interface__ holder; keeps the owning ring alive."""

    def __init__(self, ptr: int, shape, typestr: str, owner):
        self._owner = owner
        self.__cuda_array_interface__ = {
            "shape": tuple(int(s) for s in shape), "typestr": typestr,
            "data": (int(ptr), False), "version": 3, "strides": None, "stream": None,
        }


def tensor_view(ptr: int, shape, dtype, owner=None):
    """Zero-copy torch CUDA tensor over device memory at ``ptr``."""
    import torch

    name = str(dtype).replace("torch.", "")
    typestr = _TORCH_TYPESTR[name]
    t = torch.as_tensor(_CAI(ptr, shape, typestr, owner), device="cuda")
    if name == "bfloat16":
        t = t.view(torch.bfloat16)
    return t


class _HostControl:
    """POSIX shm segment holding the ring's control words (/dev/shm/<name>)."""

    def __init__(self, name: str, nbytes: int, create: bool):
        self.name = name
        self.path = f"/dev/shm/{name}"
        flags = os.O_RDWR | (os.O_CREAT | os.O_EXCL if create else 0)
        fd = os.open(self.path, flags, 0o600)
        try:
            if create:
                os.ftruncate(fd, nbytes)
            self.mm = mmap.mmap(fd, nbytes)
        finally:
            os.close(fd)
        self._buf = (ctypes.c_char * nbytes).from_buffer(self.mm)
        self.addr = ctypes.addressof(self._buf)
        self.nbytes = nbytes
        self.owner = create

    def unlink(self):
        try:
            os.unlink(self.path)
        except FileNotFoundError:
            pass


class DeviceRing:
    """``writers`` > 1: a ring of a sharded-ingest group -- slot s is complete
    once each of the writers published its shard (one ready word each)."""

    def __init__(self, slots: int, slot_bytes: int, max_consumers: int = 64,
                 device: int | None = None, control: str = "device", writers: int = 1):
        L = load()
        if device is None:
            dev = ctypes.c_int(0)
            call("tsb_get_device", ctypes.byref(dev))
            device = dev.value
        _lib.preload(device)
        h = ctypes.c_void_p()
        call("tsb_ring_create_ex", device, slots, slot_bytes, max_consumers, writers,
             ctypes.byref(h))
        self.writers = writers
        self._init(h, slots, slot_bytes, max_consumers, device, imported=False)
        self._L = L
        self.ctl = None
        if control == "host":
            nb = L.tsb_ring_control_bytes_ex(slots, max_consumers, writers)
            self.ctl = _HostControl(f"tsbc-{os.getpid()}-{id(self) & 0xFFFFFF:x}", nb, True)
            call("tsb_ring_attach_host_control", self._h, self.ctl.addr, nb, 1)
        elif control != "device":
            raise ValueError("control must be 'device' or 'host'")

    @property
    def control_name(self) -> str:
        return self.ctl.name if self.ctl is not None else "-"

    def _init(self, h, slots, slot_bytes, max_consumers, device, imported):
        self._h = h
        self.slots = slots
        self.slot_bytes = slot_bytes
        self.max_consumers = max_consumers
        self.device = device
        self.imported = imported
        self.pid = os.getpid()
        geo_slots, stride, mc = ctypes.c_int(), ctypes.c_size_t(), ctypes.c_int()
        call("tsb_ring_geometry", h, ctypes.byref(geo_slots), ctypes.byref(stride),
             ctypes.byref(mc))
        self.slot_stride = stride.value
        base = ctypes.c_void_p()
        call("tsb_ring_base_ptr", h, ctypes.byref(base))
        self.base = base.value

    @classmethod
    def import_handle(cls, handle: bytes, slots: int, slot_bytes: int, max_consumers: int,
                      control_name: str = "-", writers: int = 1):
        """Open a ring exported by another process (CUDA IPC; on this GPU, or on
        a peer GPU -- then its slots are written/read over NVLink); with a host
        control block, map the same shm segment."""
        if len(handle) != IPC_HANDLE_BYTES:
            raise ValueError("IPC handle must be 64 bytes")
        L = load()
        cur = ctypes.c_int(0)
        call("tsb_get_device", ctypes.byref(cur))
        _lib.preload(cur.value)
        buf = ctypes.create_string_buffer(handle, IPC_HANDLE_BYTES)
        h = ctypes.c_void_p()
        call("tsb_ring_import_ex", buf, slots, slot_bytes, max_consumers, writers,
             ctypes.byref(h))
        self = cls.__new__(cls)
        self._L = L
        self.writers = writers
        dev = ctypes.c_int(0)
        call("tsb_get_device", ctypes.byref(dev))
        self._init(h, slots, slot_bytes, max_consumers, dev.value, imported=True)
        self.ctl = None
        if control_name and control_name != "-":
            nb = L.tsb_ring_control_bytes_ex(slots, max_consumers, writers)
            self.ctl = _HostControl(control_name, nb, False)
            call("tsb_ring_attach_host_control", self._h, self.ctl.addr, nb, 0)
        return self

    # -- identity -----------------------------------------------------------
    def export(self) -> bytes:
        buf = ctypes.create_string_buffer(IPC_HANDLE_BYTES)
        call("tsb_ring_export", self._h, buf)
        return buf.raw

    def slot_ptr(self, slot: int) -> int:
        if not 0 <= slot < self.slots:
            raise IndexError(slot)
        return self.base + self.slot_stride * slot

    def slot_of(self, seq: int) -> int:
        return (seq - 1) % self.slots

    def view(self, slot: int, shape, dtype, byte_offset: int = 0):
        return tensor_view(self.slot_ptr(slot) + byte_offset, shape, dtype, owner=self)

    # -- device sync words ----------------------------------------------------
    def publish(self, slot: int, seq: int, stream=None) -> None:
        """Every writer's shard of the slot holds seq."""
        call("tsb_ring_publish", self._h, slot, seq, _stream(stream))

    def publish_shard(self, slot: int, writer: int, seq: int, stream=None) -> None:
        call("tsb_ring_publish_shard", self._h, slot, writer, seq, _stream(stream))

    def wait_ready(self, slot: int, seq: int, stream=None) -> None:
        call("tsb_ring_wait_ready", self._h, slot, seq, _stream(stream))

    def ack(self, consumer: int, seq: int, stream=None) -> None:
        call("tsb_ring_ack", self._h, consumer, seq, _stream(stream))

    def wait_free(self, live, seq: int, stream=None) -> None:
        if seq <= 0:
            return
        live = list(live)
        arr = (ctypes.c_int * max(1, len(live)))(*live)
        call("tsb_ring_wait_free", self._h, arr, len(live), seq, _stream(stream))

    def evict(self, consumer: int) -> None:
        call("tsb_ring_evict", self._h, consumer)

    def set_cursor(self, consumer: int, value: int) -> None:
        call("tsb_ring_set_cursor", self._h, consumer, value)

    def read_cursor(self, consumer: int) -> int:
        v = ctypes.c_uint64()
        call("tsb_ring_read_cursor", self._h, consumer, ctypes.byref(v))
        return v.value

    def read_ready(self, slot: int) -> int:
        v = ctypes.c_uint64()
        call("tsb_ring_read_ready", self._h, slot, ctypes.byref(v))
        return v.value

    # -- host-side consumer ops (host control block) ---------------------------
    def host_wait_ready(self, slot: int, seq: int, timeout_s: float = -1.0) -> None:
        """Spin on the host until the slot holds seq (no GPU channel involved)."""
        call("tsb_ring_host_wait_ready", self._h, slot, seq,
             -1 if timeout_s < 0 else int(timeout_s * 1e6))

    def host_gate(self, live, need: int, timeout_s: float = -1.0) -> bool:
        """Block until every live cursor released `need` (host control block);
        False on timeout."""
        if need <= 0:
            return True
        live = list(live)
        arr = (ctypes.c_int * max(1, len(live)))(*live)
        rc = self._L.tsb_ring_host_gate(self._h, arr, len(live), need,
                                        -1 if timeout_s < 0 else int(timeout_s * 1e6))
        if rc == _lib.TSB_ERR_STALE:
            return False
        _lib.check(rc, "tsb_ring_host_gate")
        return True

    @property
    def host_control(self) -> bool:
        return self.ctl is not None

    @property
    def cursor_words(self):
        """numpy u64 view of the release cursors in the host-shared control
        block (read-only use: the fast path of a host flow gate)."""
        v = getattr(self, "_cursor_view", None)
        if v is None:
            import numpy as np

            off = 8 * self.slots * self.writers
            v = np.frombuffer(self.ctl.mm, dtype=np.uint64, count=self.max_consumers, offset=off)
            self._cursor_view = v
        return v

    def released(self, live, need: int) -> bool:
        """True if every live cursor has released `need` (wrap-around GEQ)."""
        if not live:
            return True
        cur = self.cursor_words
        return all(((int(cur[c]) - need) & 0xFFFFFFFFFFFFFFFF) < (1 << 63) for c in live)

    def host_consume_range(self, consumer: int, seq0: int, n: int, timestamps: bool = True):
        """Native map-and-ack loop over n batches; returns fetch times (s) or None."""
        import numpy as np

        t = np.empty(max(n, 1), dtype=np.int64) if timestamps else None
        call("tsb_ring_host_consume_range", self._h, consumer, seq0, n,
             None if t is None else t.ctypes.data)
        return None if t is None else t[:n] * 1e-6

    def host_ack(self, consumer: int, seq: int) -> None:
        """Release up to seq from the host (consumer finished with the batch)."""
        call("tsb_ring_set_cursor", self._h, consumer, seq)

    def close(self) -> None:
        h, self._h = getattr(self, "_h", None), None
        if h and os.getpid() == self.pid:
            call("tsb_ring_destroy", h)
        ctl = getattr(self, "ctl", None)
        if ctl is not None and ctl.owner and os.getpid() == self.pid:
            ctl.unlink()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def sync_mode() -> str:
    return "memops" if load().tsb_ring_sync_mode() == 1 else "kernels"


def _stream(stream):
    if stream is None:
        import torch

        return _lib.stream_handle(torch.cuda.current_stream().cuda_stream)
    return _lib.stream_handle(stream)


def hold_for_stream(args, stream) -> None:
    """Keep the device buffers ``args`` points at (``args._keep``: the epoch
    order) allocated for the work enqueued on ``stream``.  The loader drops an
    epoch's order when the next epoch starts while launches that read it may
    still be queued on the producer stream (a persistent range launch, or the
    last batches of the epoch behind the slot gate); without this the caching
    allocator hands the block to the next epoch's order and those launches
    gather the wrong samples.  Recorded once per (buffer, stream)."""
    keep = getattr(args, "_keep", None)
    if not keep:
        return
    import torch

    if stream is None:
        s = torch.cuda.current_stream()
    elif isinstance(stream, torch.cuda.Stream):
        s = stream
    else:
        h = getattr(stream, "cuda_stream", stream)
        s = torch.cuda.ExternalStream(int(h.value if hasattr(h, "value") else h))
    held = args.__dict__.setdefault("_held", set())
    for t in keep:
        if isinstance(t, torch.Tensor) and t.is_cuda and (id(t), s.cuda_stream) not in held:
            t.record_stream(s)
            held.add((id(t), s.cuda_stream))


def _ev_array(events):
    if events is None:
        return None
    return (ctypes.c_void_p * len(events))(*[int(e.cuda_event) if hasattr(e, "cuda_event")
                                              else int(e) for e in events])


def produce_range(ring: DeviceRing, args, seq0: int, batch0: int, n: int, live, events=None,
                  stream=None) -> None:
    """Native producer loop: n batches of one epoch into the ring (tsb_produce_range)."""
    live = list(live)
    arr = (ctypes.c_int * max(1, len(live)))(*live)
    hold_for_stream(args, stream)
    call("tsb_produce_range", ring._h, ctypes.byref(args), seq0, batch0, n, arr, len(live),
         _ev_array(events), _stream(stream))


def consume_range(ring: DeviceRing, consumer: int, seq0: int, n: int, events=None,
                  stream=None) -> None:
    """Native consumer loop: wait_ready -> ack for n batches (tsb_consume_range)."""
    call("tsb_consume_range", ring._h, consumer, seq0, n, _ev_array(events), _stream(stream))


def produce_group(rings, local: int, args, shard: int, n_shards: int, seq0: int, batch0: int,
                  n: int, live_per_ring, stream=None) -> None:
    """Sharded ingest + fused fan-out (tsb_produce_group): writer ``shard`` of
    ``n_shards`` produces its rows of n batches of one epoch straight into the
    same slot of every ring in ``rings`` (own device's ring = rings[local],
    peers opened over CUDA IPC); the calling thread blocks on the host gate."""
    rings = list(rings)
    ptrs = (ctypes.c_void_p * len(rings))(*[r._h.value if hasattr(r._h, "value") else r._h
                                           for r in rings])
    flat = [c for lv in live_per_ring for c in lv]
    live = (ctypes.c_int * max(1, len(flat)))(*flat)
    counts = (ctypes.c_int * len(rings))(*[len(lv) for lv in live_per_ring])
    if len(live_per_ring) != len(rings):
        raise ValueError("one live list per ring")
    hold_for_stream(args, stream)
    call("tsb_produce_group", ptrs, len(rings), local, ctypes.byref(args), shard, n_shards, seq0,
         batch0, n, live, counts, _stream(stream))


def produce_group_multi(rings, args_list, locals_, devices, streams, seq0: int, batch0: int,
                        n: int, live_per_ring) -> None:
    """All writers of a single-process multi-GPU producer in one native call
    (tsb_produce_group_multi); the calling thread blocks on the host gate."""
    rings = list(rings)
    W = len(args_list)
    ptrs = (ctypes.c_void_p * len(rings))(*[r._h.value if hasattr(r._h, "value") else r._h
                                           for r in rings])
    arr = (_lib.ProduceArgs * W)(*args_list)
    loc = (ctypes.c_int * W)(*locals_)
    devs = (ctypes.c_int * W)(*devices)
    sts = (ctypes.c_void_p * W)(*[_stream(s).value for s in streams])
    flat = [c for lv in live_per_ring for c in lv]
    live = (ctypes.c_int * max(1, len(flat)))(*flat)
    counts = (ctypes.c_int * len(rings))(*[len(lv) for lv in live_per_ring])
    for a, s in zip(args_list, streams):
        hold_for_stream(a, s)
    call("tsb_produce_group_multi", ptrs, len(rings), arr, loc, devs, sts, W, seq0, batch0, n,
         live, counts)


def restage_collate(in_ring: DeviceRing, in_consumer: int, out_ring: DeviceRing, args,
                    seq0: int, n: int, live, stream=None) -> None:
    """Stage 2 of two-stage multi-GPU production (tsb_restage_collate)."""
    live = list(live)
    arr = (ctypes.c_int * max(1, len(live)))(*live)
    hold_for_stream(args, stream)
    call("tsb_restage_collate", in_ring._h, in_consumer, out_ring._h, ctypes.byref(args), seq0, n,
         arr, len(live), _stream(stream))
