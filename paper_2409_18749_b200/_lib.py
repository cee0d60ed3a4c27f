"""ctypes binding of libtsb200.so (the C ABI declared in include/tsb200.h).

There is no CPU fallback: if the CUDA library is missing or cannot be
loaded, every entry point raises ``LibraryMissing``.  Status codes map onto
the reference's exception classes (payload.py:48-61).
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import (CorruptSegmentError, DeviceError, LibraryMissing, PayloadError,
                     ResourceError, StaleHandleError)

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libtsb200.so")

TSB_OK = 0
TSB_ERR_INVALID = -1
TSB_ERR_CUDA = -2
TSB_ERR_STALE = -3
TSB_ERR_CORRUPT = -4
TSB_ERR_UNSUPPORTED = -5
IPC_HANDLE_BYTES = 64

OUT_U8, OUT_F32, OUT_BF16 = 0, 1, 2

u64, i64, i32, sz = ctypes.c_uint64, ctypes.c_int64, ctypes.c_int, ctypes.c_size_t
vp, fp = ctypes.c_void_p, ctypes.POINTER(ctypes.c_float)
pp = ctypes.POINTER(ctypes.c_void_p)

# name -> (restype, argtypes); exactly the symbols of include/tsb200.h
SIGNATURES: dict[str, tuple] = {
    "tsb_last_error": (ctypes.c_char_p, []),
    "tsb_version": (i32, []),
    "tsb_device_count": (i32, [ctypes.POINTER(i32)]),
    "tsb_set_device": (i32, [i32]),
    "tsb_get_device": (i32, [ctypes.POINTER(i32)]),
    "tsb_device_info": (i32, [i32, ctypes.POINTER(i32), ctypes.POINTER(i32), ctypes.POINTER(i32),
                              ctypes.POINTER(sz)]),
    "tsb_preload_kernels": (i32, []),
    "tsb_malloc": (i32, [pp, sz]),
    "tsb_free": (i32, [vp]),
    "tsb_host_alloc": (i32, [pp, sz]),
    "tsb_host_free": (i32, [vp]),
    "tsb_host_register": (i32, [vp, sz]),
    "tsb_host_unregister": (i32, [vp]),
    "tsb_host_device_ptr": (i32, [vp, pp]),
    "tsb_memcpy_async": (i32, [vp, vp, sz, vp]),
    "tsb_memset_async": (i32, [vp, i32, sz, vp]),
    "tsb_stream_create": (i32, [pp]),
    "tsb_stream_destroy": (i32, [vp]),
    "tsb_stream_sync": (i32, [vp]),
    "tsb_device_sync": (i32, []),
    "tsb_event_create": (i32, [pp]),
    "tsb_event_destroy": (i32, [vp]),
    "tsb_event_record": (i32, [vp, vp]),
    "tsb_event_sync": (i32, [vp]),
    "tsb_event_elapsed_ms": (i32, [vp, vp, fp]),
    "tsb_stream_wait_event": (i32, [vp, vp]),
    "tsb_enable_peer": (i32, [i32, i32]),
    "tsb_can_access_peer": (i32, [i32, i32, ctypes.POINTER(i32)]),
    "tsb_mix64": (u64, [u64]),
    "tsb_derive_key": (u64, [u64, u64, u64]),
    "tsb_permutation": (i32, [i64, u64, vp]),
    "tsb_epoch_order": (i32, [i64, u64, u64, i32, vp]),
    "tsb_fill_synthetic": (i32, [vp, vp, i64, u64, u64, i64, vp]),
    "tsb_make_store": (i32, [vp, u64, i64, i64, i64, vp]),
    "tsb_gather": (i32, [vp, vp, i64, i64, vp, vp]),
    "tsb_aug_params": (i32, [u64, u64, vp, i64, i32, i32, vp, vp]),
    "tsb_collate_augment": (i32, [vp, vp, i64, i32, i32, i32, i32, i32, u64, u64, fp, fp, i32, vp,
                                  vp, vp]),
    "tsb_crc32_workspace_bytes": (sz, []),
    "tsb_crc32": (i32, [vp, sz, vp, vp, vp]),
    "tsb_ring_create": (i32, [i32, i32, sz, i32, pp]),
    "tsb_ring_export": (i32, [vp, vp]),
    "tsb_ring_import": (i32, [vp, i32, sz, i32, pp]),
    "tsb_ring_destroy": (i32, [vp]),
    "tsb_ring_slot_ptr": (i32, [vp, i32, pp]),
    "tsb_ring_base_ptr": (i32, [vp, pp]),
    "tsb_ring_geometry": (i32, [vp, ctypes.POINTER(i32), ctypes.POINTER(sz), ctypes.POINTER(i32)]),
    "tsb_ring_publish": (i32, [vp, i32, u64, vp]),
    "tsb_ring_wait_ready": (i32, [vp, i32, u64, vp]),
    "tsb_ring_ack": (i32, [vp, i32, u64, vp]),
    "tsb_ring_wait_free": (i32, [vp, ctypes.POINTER(i32), i32, u64, vp]),
    "tsb_ring_evict": (i32, [vp, i32]),
    "tsb_ring_set_cursor": (i32, [vp, i32, u64]),
    "tsb_ring_read_cursor": (i32, [vp, i32, ctypes.POINTER(u64)]),
    "tsb_ring_read_ready": (i32, [vp, i32, ctypes.POINTER(u64)]),
    "tsb_ring_sync_mode": (i32, []),
    "tsb_ring_control_bytes": (sz, [i32, i32]),
    "tsb_ring_attach_host_control": (i32, [vp, vp, sz, i32]),
    "tsb_ring_host_wait_ready": (i32, [vp, i32, u64, i64]),
    "tsb_ring_host_gate": (i32, [vp, ctypes.POINTER(i32), i32, u64, i64]),
    "tsb_ring_host_consume_range": (i32, [vp, i32, u64, i32, vp]),
    "tsb_ring_create_ex": (i32, [i32, i32, sz, i32, i32, pp]),
    "tsb_ring_import_ex": (i32, [vp, i32, sz, i32, i32, pp]),
    "tsb_ring_writers": (i32, [vp, ctypes.POINTER(i32)]),
    "tsb_ring_publish_shard": (i32, [vp, i32, i32, u64, vp]),
    "tsb_ring_control_bytes_ex": (sz, [i32, i32, i32]),
    "tsb_fanout": (i32, [vp, pp, i32, sz, vp]),
    "tsb_collate_augment_fanout": (i32, [vp, vp, i64, i32, i32, i32, i32, i32, u64, u64, fp, fp,
                                         i32, pp, i32, vp]),
    "tsb_rebatch_gather": (i32, [vp, i64, i64, i64, i64, vp, vp]),
    "tsb_rebatch_window": (i32, [pp, i32, i64, i64, i64, i64, i64, vp, vp]),
    "tsb_ingest_create": (i32, [i32, i64, i64, i32, pp]),
    "tsb_ingest_destroy": (i32, [vp]),
    "tsb_ingest_batch_api": (i32, [vp, ctypes.POINTER(i32)]),
    "tsb_ingest_bytes": (i32, [vp, ctypes.POINTER(ctypes.c_uint64)]),
    "tsb_jpeg_available": (i32, [ctypes.POINTER(i32)]),
    "tsb_jpeg_create": (i32, [i32, i64, i32, i32, i32, pp]),
    "tsb_jpeg_backend": (i32, [vp, ctypes.POINTER(i32)]),
    "tsb_jpeg_attach_store": (i32, [vp, pp, ctypes.POINTER(sz), i64]),
    "tsb_jpeg_decode": (i32, [vp, vp, i64, vp, vp]),
    "tsb_jpeg_destroy": (i32, [vp]),
}

class ProduceArgs(ctypes.Structure):
    """Mirror of tsb_produce_args (include/tsb200.h)."""
    _fields_ = [
        ("mode", ctypes.c_int), ("src", ctypes.c_void_p), ("d_order", ctypes.c_void_p),
        ("batch_size", ctypes.c_int64), ("sample_bytes", ctypes.c_int64),
        ("h", ctypes.c_int), ("w", ctypes.c_int), ("c", ctypes.c_int), ("pad", ctypes.c_int),
        ("flip", ctypes.c_int), ("out_kind", ctypes.c_int), ("seed", ctypes.c_uint64),
        ("epoch", ctypes.c_uint64), ("scale", ctypes.c_float * 4), ("bias", ctypes.c_float * 4),
        ("with_target", ctypes.c_int), ("input_bytes", ctypes.c_int64),
        ("d_crc", ctypes.c_void_p), ("wait_stride", ctypes.c_int), ("gate", ctypes.c_int),
        ("ingest", ctypes.c_void_p), ("h_order", ctypes.c_void_p), ("persistent", ctypes.c_int),
        ("chain", ctypes.c_int),
        ("jpeg", ctypes.c_void_p),
        ("h_crc", ctypes.c_void_p), ("crc_fused", ctypes.c_void_p),
        ("order_epochs", ctypes.c_int64), ("epoch_len", ctypes.c_int64),
        ("order_stride", ctypes.c_int64),
    ]


GATE_DEVICE, GATE_HOST = 0, 1


class Msg(ctypes.Structure):
    """Mirror of tsb_msg (include/tsb200.h)."""
    _fields_ = [
        ("kind", ctypes.c_uint8), ("consumer_id", ctypes.c_uint64),
        ("protocol_version", ctypes.c_uint16), ("device", ctypes.c_int16),
        ("batch_size", ctypes.c_uint32), ("epoch", ctypes.c_uint32),
        ("epoch_len", ctypes.c_uint64), ("next_batch_index", ctypes.c_uint64),
        ("buffer_depth", ctypes.c_uint16), ("admitted", ctypes.c_uint8),
        ("batch_index", ctypes.c_uint64), ("monotonic_millis", ctypes.c_uint64),
        ("name_len", ctypes.c_uint16), ("segment_name", ctypes.c_char * 256),
        ("byte_len", ctypes.c_uint64), ("dtype", ctypes.c_uint8), ("ndim", ctypes.c_uint8),
        ("shape", ctypes.c_uint64 * 8), ("checksum", ctypes.c_uint32),
    ]


SRC_AUGMENT, SRC_GATHER, SRC_SYNTHETIC = 0, 1, 2

SIGNATURES["tsb_produce_range"] = (i32, [vp, ctypes.POINTER(ProduceArgs), u64, i64, i32,
                                         ctypes.POINTER(i32), i32, pp, vp])
SIGNATURES["tsb_consume_range"] = (i32, [vp, i32, u64, i32, pp, vp])
SIGNATURES["tsb_restage_collate"] = (i32, [vp, i32, vp, ctypes.POINTER(ProduceArgs), u64, i32,
                                           ctypes.POINTER(i32), i32, vp])
SIGNATURES["tsb_produce_group_multi"] = (i32, [pp, i32, ctypes.POINTER(ProduceArgs),
                                               ctypes.POINTER(i32), ctypes.POINTER(i32), pp, i32,
                                               u64, i64, i32, ctypes.POINTER(i32),
                                               ctypes.POINTER(i32)])
class HubEvent(ctypes.Structure):
    """Mirror of tsb_hub_event (include/tsb200.h)."""
    _fields_ = [("kind", ctypes.c_uint8), ("consumer_id", ctypes.c_uint64),
                ("epoch", ctypes.c_uint32), ("batch_index", ctypes.c_uint64),
                ("t_us", ctypes.c_int64), ("fd", ctypes.c_int32)]


SIGNATURES["tsb_hub_create"] = (i32, [pp])
SIGNATURES["tsb_hub_add"] = (i32, [vp, i32, u64, vp, sz])
SIGNATURES["tsb_hub_remove"] = (i32, [vp, i32])
SIGNATURES["tsb_hub_drain"] = (i32, [vp, ctypes.POINTER(HubEvent), i32, ctypes.POINTER(i32)])
SIGNATURES["tsb_hub_broadcast"] = (i32, [ctypes.POINTER(i32), i32, vp, sz, ctypes.POINTER(i32)])
SIGNATURES["tsb_hub_destroy"] = (i32, [vp])
SIGNATURES["tsb_hub_set_epoch_len"] = (i32, [vp, u64])
SIGNATURES["tsb_hub_set_acked"] = (i32, [vp, u64, u64])
SIGNATURES["tsb_hub_read_acked"] = (i32, [vp, u64, ctypes.POINTER(u64)])
SIGNATURES["tsb_hub_wait_acked"] = (i32, [vp, ctypes.POINTER(u64), i32, u64, i64])
SIGNATURES["tsb_hub_drift_max"] = (i32, [vp, ctypes.POINTER(u64)])
SIGNATURES["tsb_facade_create"] = (i32, [pp])
SIGNATURES["tsb_facade_destroy"] = (i32, [vp])
SIGNATURES["tsb_facade_set_batch"] = (i32, [vp, vp, vp, ctypes.POINTER(ProduceArgs), vp, i32, u64,
                                            ctypes.c_char_p, u64, vp, vp, pp, i32])
SIGNATURES["tsb_facade_set_consumers"] = (i32, [vp, ctypes.POINTER(u64), i32, ctypes.POINTER(i32),
                                                i32, ctypes.POINTER(i32), i32])
SIGNATURES["tsb_facade_produce"] = (i32, [vp, u64, i64, i32, i64])
SIGNATURES["tsb_facade_step"] = (i32, [vp, u64, i64, i32, i64, u64, ctypes.c_uint32, u64, i32,
                                       ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(i32)])
SIGNATURES["tsb_facade_announce"] = (i32, [vp, u64, ctypes.c_uint32, u64, i32,
                                           ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(i32)])
SIGNATURES["tsb_wire_encode"] = (i32, [ctypes.POINTER(Msg), vp, sz, ctypes.POINTER(sz)])
SIGNATURES["tsb_wire_decode"] = (i32, [vp, sz, ctypes.POINTER(Msg), ctypes.POINTER(sz)])
SIGNATURES["tsb_produce_group"] = (i32, [pp, i32, i32, ctypes.POINTER(ProduceArgs), i32, i32, u64,
                                         i64, i32, ctypes.POINTER(i32), ctypes.POINTER(i32), vp])

_lib = None
_lock = threading.Lock()


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libtsb200.so; raises LibraryMissing (never falls back to CPU)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise LibraryMissing(
                f"{path} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        try:
            lib = ctypes.CDLL(path)
        except OSError as exc:
            raise LibraryMissing(f"cannot load {path}: {exc}") from exc
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def last_error() -> str:
    return (load().tsb_last_error() or b"").decode(errors="replace")


_EXC = {
    TSB_ERR_INVALID: ValueError,
    TSB_ERR_CUDA: ResourceError,
    TSB_ERR_STALE: StaleHandleError,
    TSB_ERR_CORRUPT: CorruptSegmentError,
    TSB_ERR_UNSUPPORTED: DeviceError,
}


def check(rc: int, what: str = "") -> None:
    if rc != TSB_OK:
        exc = _EXC.get(rc, PayloadError)
        raise exc(f"{what}: {last_error()}" if what else last_error())


def call(name: str, *args):
    rc = getattr(load(), name)(*args)
    check(rc, name)


def stream_handle(stream) -> ctypes.c_void_p:
    """Accept None, an int handle, a torch.cuda.Stream or anything with .cuda_stream."""
    if stream is None:
        return ctypes.c_void_p(0)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    h = getattr(stream, "cuda_stream", None)
    if h is not None:
        return ctypes.c_void_p(int(h))
    return ctypes.c_void_p(int(stream))


def exported_symbols() -> list[str]:
    return list(SIGNATURES)


_preloaded: set = set()


def preload(device: int) -> None:
    """Eager-load the library's kernels in `device`'s context (once)."""
    if device in _preloaded:
        return
    import torch

    with torch.cuda.device(device):
        call("tsb_preload_kernels")
    _preloaded.add(device)
