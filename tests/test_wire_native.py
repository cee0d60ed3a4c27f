"""Native C++ control-plane codec (tsb_wire_encode/decode) on CPU: the frozen
frames the reference produced (tests/test_wire.py:56-85,
ftests/test_abi.py:9-52) encode byte-identically, decode back, and agree with
the Python codec on random messages, including the bf16 DType and Join v2."""

import ctypes

import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2409_18749_b200 import _lib
from paper_2409_18749_b200.wire import (Ack, Announce, Bye, EpochEnd, EpochStart, Heartbeat, Join,
                                        Shutdown, Welcome, decode, encode)

KINDS = {Join: 1, Welcome: 2, Announce: 3, Ack: 4, Heartbeat: 5, EpochStart: 6, EpochEnd: 7,
         Bye: 8, Shutdown: 9}


def to_msg(m) -> _lib.Msg:
    c = _lib.Msg()
    c.kind = KINDS[type(m)]
    c.device = -1
    for f in getattr(m, "__dataclass_fields__", {}):
        v = getattr(m, f)
        if f == "segment_name":
            b = v.encode()
            c.name_len = len(b)
            c.segment_name = b
        elif f == "shape":
            c.ndim = len(v)
            for i, d in enumerate(v):
                c.shape[i] = d
        else:
            setattr(c, f, int(v))
    return c


def native_encode(m) -> bytes:
    buf = ctypes.create_string_buffer(70000)
    n = ctypes.c_size_t()
    _lib.call("tsb_wire_encode", ctypes.byref(to_msg(m)), buf, len(buf), ctypes.byref(n))
    return buf.raw[:n.value]


def native_decode(frame: bytes):
    m = _lib.Msg()
    off = ctypes.c_size_t()
    rc = _lib.load().tsb_wire_decode(frame, len(frame), ctypes.byref(m), ctypes.byref(off))
    return rc, m, off.value


def test_golden_frames_roundtrip(golden):
    for name, hexframe in list(golden["frames"].items()) + list(golden["facade_frames"].items()):
        frame = bytes.fromhex(hexframe)
        msg = decode(frame)  # the Python codec (pinned by tests/test_wire.py)
        assert native_encode(msg) == frame, name
        rc, m, _ = native_decode(frame)
        assert rc == 0 and m.kind == KINDS[type(msg)], name


def test_extensions_and_errors():
    for m in (Join(7, 2, 3, 128), Join(9, 2),
              Announce(1, 2, "tsb1:ab:3:xyz", 8, 5, (2, 2), 7)):  # bf16 dtype code 5
        assert native_encode(m) == encode(m)
    rc, m, _ = native_decode(encode(Join(7, 2, 3, 128)))
    assert rc == 0 and (m.device, m.batch_size) == (3, 128)
    assert native_decode(b"\x01\x00")[0] == _lib.TSB_ERR_CORRUPT            # truncated prefix
    assert native_decode(b"\x00\x00\x00\x00")[0] == _lib.TSB_ERR_CORRUPT    # no kind byte
    assert native_decode(b"\x01\x00\x00\x00\x0a")[0] == _lib.TSB_ERR_CORRUPT  # unknown kind
    f = bytearray(encode(Ack(1, 2, 3)))
    f[0] += 1
    assert native_decode(bytes(f) + b"\x00")[0] == _lib.TSB_ERR_CORRUPT   # trailing byte
    with pytest.raises(ValueError):
        native_encode(Join(1, 1, 0, 0))  # v2 fields on a v1 Join


names = st.text(alphabet=st.characters(min_codepoint=33, max_codepoint=126), min_size=1,
                max_size=60)
u32 = st.integers(0, 2**32 - 1)
u64 = st.integers(0, 2**64 - 1)


@st.composite
def announces(draw):
    shape = tuple(draw(st.lists(st.integers(0, 9), max_size=4)))
    dt = draw(st.integers(0, 5))
    n = (1, 4, 8, 4, 8, 2)[dt]
    for d in shape:
        n *= d
    return Announce(draw(u32), draw(u64), draw(names), n, dt, shape, draw(u32))


msgs = st.one_of(
    st.builds(Join, u64), st.builds(Join, u64, st.just(2), st.integers(-1, 32767), u32),
    st.builds(Welcome, u64, u32, st.integers(1, 2**64 - 1), u64, st.integers(0, 65535),
              st.integers(0, 2)),
    announces(), st.builds(Ack, u64, u32, u64), st.builds(Heartbeat, u64, u64),
    st.builds(EpochStart, u32, st.integers(1, 2**64 - 1)), st.builds(EpochEnd, u32),
    st.builds(Bye, u64), st.just(Shutdown()))


@settings(max_examples=300, deadline=None)
@given(msgs)
def test_native_matches_python_codec(m):
    frame = encode(m)
    assert native_encode(m) == frame
    rc, c, _ = native_decode(frame)
    assert rc == 0
    assert native_encode(decode(frame)) == frame
