"""Control-plane codec, byte-compatible with the reference wire format.

Frame: ``u32le body_len | u8 kind | body`` (body_len counts the kind byte);
integers little-endian fixed width, strings ``u16 len | utf-8``.  Kinds
1..9 = Join, Welcome, Announce, Ack, Heartbeat, EpochStart, EpochEnd, Bye,
Shutdown (reference: pkg/src/batchsocket/wire.py:1-11,77-156,199-341;
facade codec pkg/frontend/src/sharedloader/abi.py:131-226).  Golden frames
produced by the reference are pinned in tests/test_wire.py.

Additions (behind the same frame format):
* ``DType.BF16 = 5`` (2 bytes) -- the reference's closed set is 0..4
  (wire.py:49-74); only this implementation emits it.
* device-slot URIs in ``Announce.segment_name`` (see ``segment.py``).
* Join v2 (``protocol_version == 2``): the v1 body ``u64 consumer_id | u16
  version`` followed by ``i16 device | u32 batch_size`` -- the consumer's GPU
  (which device ring it maps) and its own batch size (heterogeneous
  consumers, 0 = the producer's).  v1 Joins (the reference's) decode as
  before, with device = -1 and batch_size = 0.
"""

from __future__ import annotations

import struct
import zlib
from dataclasses import dataclass
from enum import IntEnum

PROTOCOL_VERSION = 1
JOIN_V2 = 2
SUPPORTED_VERSIONS = (PROTOCOL_VERSION, JOIN_V2)
MAX_FRAME_BODY = 65536
MAX_SEGMENT_NAME = 255
MAX_NDIM = 8

ADMIT_WAIT, ADMIT_RUBBERBAND, ADMIT_IMMEDIATE = 0, 1, 2


class EncodeError(ValueError):
    """Message violates a wire invariant."""


class DecodeError(ValueError):
    """Frame bytes are not a valid message; carries the failing byte offset."""

    def __init__(self, offset: int, cause: str):
        super().__init__(f"decode error at offset {offset}: {cause}")
        self.offset = offset
        self.cause = cause


class DType(IntEnum):
    U8 = 0
    I32 = 1
    I64 = 2
    F32 = 3
    F64 = 4
    BF16 = 5  # extension (device batches)

    @property
    def size(self) -> int:
        return (1, 4, 8, 4, 8, 2)[int(self)]

    @property
    def numpy_name(self) -> str:
        return ("uint8", "int32", "int64", "float32", "float64", "bfloat16")[int(self)]

    @property
    def torch_name(self) -> str:
        return ("uint8", "int32", "int64", "float32", "float64", "bfloat16")[int(self)]


def dtype_of(obj) -> DType:
    """DType of a numpy array / torch tensor (TypeError if unsupported)."""
    name = str(getattr(obj, "dtype", obj)).replace("torch.", "")
    table = {"uint8": DType.U8, "int32": DType.I32, "int64": DType.I64,
             "float32": DType.F32, "float64": DType.F64, "bfloat16": DType.BF16}
    if name not in table:
        raise TypeError(f"unsupported array dtype: {name}")
    return table[name]


# -- messages ---------------------------------------------------------------

@dataclass(frozen=True)
class Join:
    consumer_id: int
    protocol_version: int = PROTOCOL_VERSION
    device: int = -1        # v2 only
    batch_size: int = 0     # v2 only


@dataclass(frozen=True)
class Welcome:
    consumer_id: int
    epoch: int
    epoch_len: int
    next_batch_index: int
    buffer_depth: int
    admitted: int


@dataclass(frozen=True)
class Announce:
    epoch: int
    batch_index: int
    segment_name: str
    byte_len: int
    dtype: int
    shape: tuple
    checksum: int


@dataclass(frozen=True)
class Ack:
    consumer_id: int
    epoch: int
    batch_index: int


@dataclass(frozen=True)
class Heartbeat:
    consumer_id: int
    monotonic_millis: int


@dataclass(frozen=True)
class EpochStart:
    epoch: int
    epoch_len: int


@dataclass(frozen=True)
class EpochEnd:
    epoch: int


@dataclass(frozen=True)
class Bye:
    consumer_id: int


@dataclass(frozen=True)
class Shutdown:
    pass


# kind -> (class, struct of the fixed body or None for Announce)
_FIXED = {
    1: (Join, struct.Struct("<QH")),
    2: (Welcome, struct.Struct("<QIQQHB")),
    4: (Ack, struct.Struct("<QIQ")),
    5: (Heartbeat, struct.Struct("<QQ")),
    6: (EpochStart, struct.Struct("<IQ")),
    7: (EpochEnd, struct.Struct("<I")),
    8: (Bye, struct.Struct("<Q")),
    9: (Shutdown, struct.Struct("<")),
}
ANNOUNCE_KIND = 3
KIND = {cls: k for k, (cls, _) in _FIXED.items()}
KIND[Announce] = ANNOUNCE_KIND
_HEAD = struct.Struct("<IB")
_JOIN_V2 = struct.Struct("<QHhI")


def checksum(data) -> int:
    """CRC-32/IEEE of a host buffer (wire.py:170-172)."""
    return zlib.crc32(data) & 0xFFFFFFFF


def _announce_problem(msg: Announce) -> str | None:
    name = msg.segment_name.encode("utf-8")
    if not name:
        return "empty segment_name"
    if len(name) > MAX_SEGMENT_NAME:
        return f"segment_name is {len(name)} bytes (max {MAX_SEGMENT_NAME})"
    if len(msg.shape) > MAX_NDIM:
        return f"ndim {len(msg.shape)} exceeds {MAX_NDIM}"
    try:
        dt = DType(msg.dtype)
    except ValueError:
        return f"unknown dtype code {msg.dtype}"
    n = dt.size
    for d in msg.shape:
        n *= d
    if n != msg.byte_len:
        return "shape/dtype product does not match byte_len"
    return None


def encode(msg) -> bytes:
    kind = KIND.get(type(msg))
    if kind is None:
        raise EncodeError(f"not a control message: {type(msg).__name__}")
    if kind == ANNOUNCE_KIND:
        bad = _announce_problem(msg)
        if bad:
            raise EncodeError(bad)
        name = msg.segment_name.encode("utf-8")
        nd = len(msg.shape)
        body = struct.pack(f"<IQH{len(name)}sQBB{nd}QI", msg.epoch, msg.batch_index, len(name),
                           name, msg.byte_len, int(msg.dtype), nd, *msg.shape, msg.checksum)
    elif kind == 1 and msg.protocol_version >= JOIN_V2:
        if not (-1 <= msg.device < 32768 and 0 <= msg.batch_size < (1 << 32)):
            raise EncodeError("Join v2 device/batch_size out of range")
        body = _JOIN_V2.pack(msg.consumer_id, msg.protocol_version, msg.device, msg.batch_size)
    else:
        cls, st = _FIXED[kind]
        if cls is EpochStart and msg.epoch_len <= 0:
            raise EncodeError("epoch_len must be > 0")
        if cls is Join and (msg.device != -1 or msg.batch_size != 0):
            raise EncodeError("device/batch_size need protocol_version >= 2")
        fields = ("consumer_id", "protocol_version") if cls is Join else cls.__dataclass_fields__
        body = st.pack(*(getattr(msg, f) for f in fields))
    return _HEAD.pack(len(body) + 1, kind) + body


def decode(frame: bytes):
    """Decode exactly one complete frame (length prefix included)."""
    if len(frame) < 4:
        raise DecodeError(0, "truncated length prefix")
    (length,) = struct.unpack_from("<I", frame, 0)
    if length == 0:
        raise DecodeError(4, "missing kind byte (zero-length body)")
    if length > MAX_FRAME_BODY:
        raise DecodeError(0, f"declared length {length} exceeds {MAX_FRAME_BODY}")
    if len(frame) != 4 + length:
        raise DecodeError(4, f"frame is {len(frame)} bytes, declared {4 + length}")
    kind = frame[4]
    end = 4 + length
    if kind == ANNOUNCE_KIND:
        msg, used = _decode_announce(frame)
    elif kind == 1 and length - 1 == _JOIN_V2.size:
        cid, ver, dev, bsz = _JOIN_V2.unpack_from(frame, 5)
        if ver < JOIN_V2:
            raise DecodeError(13, f"Join v{ver} body carries v2 fields")
        msg, used = Join(cid, ver, dev, bsz), 5 + _JOIN_V2.size
    elif kind in _FIXED:
        cls, st = _FIXED[kind]
        if 5 + st.size > end:
            raise DecodeError(5, f"truncated {cls.__name__}")
        vals = st.unpack_from(frame, 5)
        if cls is Welcome:
            if vals[2] == 0:
                raise DecodeError(13, "epoch_len must be > 0")
            if vals[5] > 2:
                raise DecodeError(5 + st.size - 1, f"unknown admitted code {vals[5]}")
        if cls is EpochStart and vals[1] == 0:
            raise DecodeError(9, "epoch_len must be > 0")
        msg, used = cls(*vals), 5 + st.size
    else:
        raise DecodeError(4, f"unknown message kind {kind}")
    if used != end:
        raise DecodeError(used, f"{end - used} trailing bytes in body")
    return msg


def _decode_announce(frame: bytes):
    off = 5

    def take(fmt: str, what: str):
        nonlocal off
        n = struct.calcsize(fmt)
        if off + n > len(frame):
            raise DecodeError(off, f"truncated {what}")
        v = struct.unpack_from(fmt, frame, off)
        off += n
        return v

    epoch, batch_index = take("<IQ", "Announce")
    (nlen,) = take("<H", "segment_name length")
    if nlen > MAX_SEGMENT_NAME:
        raise DecodeError(off - 2, f"segment_name is {nlen} bytes (max {MAX_SEGMENT_NAME})")
    if off + nlen > len(frame):
        raise DecodeError(off, "truncated segment_name")
    try:
        name = frame[off:off + nlen].decode("utf-8")
    except UnicodeDecodeError as exc:
        raise DecodeError(off, f"segment_name is not UTF-8: {exc}") from None
    off += nlen
    byte_len, code, ndim = take("<QBB", "Announce tail")
    if ndim > MAX_NDIM:
        raise DecodeError(off - 1, f"ndim {ndim} exceeds {MAX_NDIM}")
    shape = take(f"<{ndim}Q", "shape") if ndim else ()
    (crc,) = take("<I", "checksum")
    try:
        dt = DType(code)
    except ValueError:
        raise DecodeError(off - 8 * ndim - 6, f"unknown dtype code {code}") from None
    msg = Announce(epoch, batch_index, name, byte_len, dt, tuple(shape), crc)
    bad = _announce_problem(msg)
    if bad:
        raise DecodeError(5, bad)
    return msg, off


class FrameDecoder:
    """Incremental decoder: feed arbitrary chunks, get complete messages."""

    def __init__(self):
        self._buf = bytearray()

    def feed(self, data: bytes) -> list:
        self._buf += data
        out = []
        while len(self._buf) >= 4:
            (length,) = struct.unpack_from("<I", self._buf, 0)
            if length > MAX_FRAME_BODY:
                raise DecodeError(0, f"declared length {length} exceeds {MAX_FRAME_BODY}")
            if len(self._buf) < 4 + length:
                break
            frame = bytes(self._buf[:4 + length])
            del self._buf[:4 + length]
            out.append(decode(frame))
        return out

    @property
    def pending_bytes(self) -> int:
        return len(self._buf)

    def take_pending(self) -> bytes:
        """Bytes received past the last complete frame (and forget them)."""
        b = bytes(self._buf)
        self._buf.clear()
        return b


# reference-compatible aliases
encode_message = encode
decode_message = decode
