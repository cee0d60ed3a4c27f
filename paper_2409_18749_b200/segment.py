"""Segment header ABI and device-slot names.

The reference writes each batch as ``80-byte header || payload`` into a POSIX
shm segment (payload.py:3-21,42).  Here the payload lives in a device ring
slot, and the *same* 80-byte header (bit-identical layout, "TSKB", version 1)
travels base64-encoded inside ``Announce.segment_name`` together with the
slot index, so the consumer gets the header without a device read:

    tsb1:<ring_id>:<slot>:<b64(80-byte header)>           (data announce)

The ring itself (CUDA-IPC handle + geometry) is described once per consumer
by a private "ring descriptor" announce with ``epoch == RING_EPOCH``
(0xFFFFFFFF), ``batch_index`` = the consumer's device cursor index and

    tsbr:<ring_id>:<pid>:<device>:<slots>:<slot_bytes>:<max_consumers>:<ctl>:<b64(ipc)>
    tsbr2:<...same...>:<ctl>:<writers>:<per_slot>:<samples>:<b64(ipc)>

(v2: ``writers`` ready words per slot -- sharded ingest; ``per_slot`` =
producer batch size and ``samples`` = samples per epoch, for consumers that
rebatch to their own batch size; the ring is the one on the consumer's GPU).

Reference consumers ignore it (epoch mismatch, sl/loader.py:155-156).
Pair encoding (input+target in one blob) follows sl/abi.py:27-31,291-308:
reserved = "PR01" | in_dtype u8 | in_ndim u8 | tg_dtype u8 | tg_ndim u8 |
input_byte_len u64, and the unused shape slots hold input then target dims.
"""

from __future__ import annotations

import base64
import struct
from dataclasses import dataclass

from .wire import DType

HEADER_SIZE = 80
MAGIC = b"TSKB"
SEGMENT_VERSION = 1
MAX_NDIM = 8
PAIR_MAGIC = b"PR01"
RING_EPOCH = 0xFFFFFFFF

_HEADER = struct.Struct("<4sHBBIIQQ8I16s")
assert _HEADER.size == HEADER_SIZE
_PAIR = struct.Struct("<4sBBBBQ")


@dataclass(frozen=True)
class SegmentHeader:
    epoch: int
    batch_index: int
    dtype: int
    shape: tuple
    byte_len: int
    checksum: int
    raw_slots: tuple
    reserved: bytes


def pack_header(epoch: int, batch_index: int, dtype: int, shape, byte_len: int, crc: int,
                reserved: bytes = b"", extra_slots=()) -> bytes:
    """payload.py:220-233 / sl/abi.py:244-251 layout."""
    slots = [int(d) for d in shape] + [int(d) for d in extra_slots]
    if len(shape) > MAX_NDIM or len(slots) > MAX_NDIM:
        raise ValueError("shape and extra slots exceed the 8 header slots")
    if any(d < 0 or d > 0xFFFFFFFF for d in slots):
        raise ValueError(f"shape {tuple(shape)} has a dimension outside u32 range")
    if len(reserved) > 16:
        raise ValueError("reserved region is 16 bytes")
    slots += [0] * (MAX_NDIM - len(slots))
    return _HEADER.pack(MAGIC, SEGMENT_VERSION, int(dtype), len(shape), epoch, crc, batch_index,
                        byte_len, *slots, reserved.ljust(16, b"\x00"))


def unpack_header(buf: bytes) -> SegmentHeader:
    from .errors import CorruptSegmentError

    if len(buf) < HEADER_SIZE:
        raise CorruptSegmentError(f"header is {len(buf)} bytes, below {HEADER_SIZE}")
    magic, ver, dt, ndim, epoch, crc, bidx, blen, *rest = _HEADER.unpack_from(buf, 0)
    if magic != MAGIC:
        raise CorruptSegmentError(f"bad magic {magic!r}")
    if ver != SEGMENT_VERSION:
        raise CorruptSegmentError(f"segment version {ver} != {SEGMENT_VERSION}")
    if ndim > MAX_NDIM:
        raise CorruptSegmentError(f"ndim {ndim} exceeds {MAX_NDIM}")
    try:
        dtype = DType(dt)
    except ValueError:
        raise CorruptSegmentError(f"unknown dtype code {dt}") from None
    slots = tuple(int(d) for d in rest[:MAX_NDIM])
    shape = slots[:ndim]
    n = dtype.size
    for d in shape:
        n *= d
    if n != blen:
        raise CorruptSegmentError(f"header shape {shape} x {dtype.name} implies {n} bytes, "
                                  f"header says {blen}")
    return SegmentHeader(epoch, bidx, dtype, shape, blen, crc, slots, rest[MAX_NDIM])


def pack_pair_reserved(in_dtype: int, in_ndim: int, tg_dtype: int, tg_ndim: int,
                       input_byte_len: int) -> bytes:
    return _PAIR.pack(PAIR_MAGIC, in_dtype, in_ndim, tg_dtype, tg_ndim, input_byte_len)


def unpack_pair(h: SegmentHeader):
    """((in_dtype, in_shape), (tg_dtype, tg_shape), input_byte_len) or None."""
    if h.reserved[:4] != PAIR_MAGIC:
        return None
    _, idt, ind, tdt, tnd, inb = _PAIR.unpack_from(h.reserved, 0)
    s = h.raw_slots
    return (idt, tuple(s[1:1 + ind])), (tdt, tuple(s[1 + ind:1 + ind + tnd])), inb


def _b64(b: bytes) -> str:
    return base64.b64encode(b).decode("ascii")


def slot_name(ring_id: int, slot: int, header: bytes) -> str:
    name = f"tsb1:{ring_id:x}:{slot}:{_b64(header)}"
    assert len(name) <= 255
    return name


def parse_slot_name(name: str):
    """-> (ring_id, slot, header bytes) or None if not a device-slot name."""
    if not name.startswith("tsb1:"):
        return None
    _, rid, slot, hb = name.split(":", 3)
    return int(rid, 16), int(slot), base64.b64decode(hb)


@dataclass(frozen=True)
class RingDescriptor:
    ring_id: int
    pid: int
    device: int
    slots: int
    slot_bytes: int
    max_consumers: int
    ipc_handle: bytes
    control: str = "-"  # host-shared control block (shm name) or "-" (device words)
    writers: int = 1
    per_slot: int = 0   # producer batch size (samples per slot); 0 = unknown
    samples: int = 0    # samples per epoch; 0 = unknown

    def name(self) -> str:
        head = (f"{self.ring_id:x}:{self.pid}:{self.device}:{self.slots}:{self.slot_bytes}:"
                f"{self.max_consumers}:{self.control}")
        if self.writers == 1 and not self.per_slot and not self.samples:
            n = f"tsbr:{head}:{_b64(self.ipc_handle)}"
        else:
            n = (f"tsbr2:{head}:{self.writers}:{self.per_slot}:{self.samples}:"
                 f"{_b64(self.ipc_handle)}")
        assert len(n) <= 255
        return n

    @classmethod
    def parse(cls, name: str) -> "RingDescriptor | None":
        if name.startswith("tsbr:"):
            _, rid, pid, dev, slots, sb, mc, ctl, h = name.split(":", 8)
            return cls(int(rid, 16), int(pid), int(dev), int(slots), int(sb), int(mc),
                       base64.b64decode(h), ctl)
        if name.startswith("tsbr2:"):
            _, rid, pid, dev, slots, sb, mc, ctl, wr, ps, ns, h = name.split(":", 11)
            return cls(int(rid, 16), int(pid), int(dev), int(slots), int(sb), int(mc),
                       base64.b64decode(h), ctl, int(wr), int(ps), int(ns))
        return None
