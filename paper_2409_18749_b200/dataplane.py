"""Python face of the device data-plane kernels (thin wrappers over the C ABI).

Device buffers are passed as torch CUDA tensors (PyTorch is the plumbing for
device memory and streams) or raw integer device pointers; the stream is a
torch stream / raw handle / None (= torch's current stream).  Every call
launches hand-written sm_100a kernels from libtsb200.so; nothing here runs
on the CPU except the once-per-epoch Fisher-Yates shuffle, which the
reference also runs sequentially (kernels.py:123-140).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._lib import OUT_BF16, OUT_F32, OUT_U8, call, load

GAMMA = 0x9E3779B97F4A7C15
SHUFFLE_DOMAIN = 0x53485546  # pipeline.py:25
M64 = (1 << 64) - 1
IMAGENET_MEAN = (0.485, 0.456, 0.406)
IMAGENET_STD = (0.229, 0.224, 0.225)


def ptr(x) -> int:
    """Device (or pinned-host) address of a tensor / pointer-like."""
    if x is None:
        return 0
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return int(x.data_ptr())
    if hasattr(x, "ptr"):
        return int(x.ptr)
    if isinstance(x, np.ndarray):
        return int(x.ctypes.data)
    raise TypeError(f"cannot take the address of {type(x).__name__}")


def current_stream(stream=None):
    if stream is not None:
        return _lib.stream_handle(stream)
    import torch

    return _lib.stream_handle(torch.cuda.current_stream().cuda_stream)


# -- RNG + shuffle (host native, kernels.py / pipeline.py) -------------------

def mix64(x: int) -> int:
    return int(load().tsb_mix64(x & M64))


def derive_key(seed: int, epoch: int, index: int) -> int:
    return int(load().tsb_derive_key(seed & M64, epoch & M64, index & M64))


def permutation(n: int, key: int) -> np.ndarray:
    if n < 0:
        raise ValueError("n must be >= 0")
    out = np.empty(n, dtype=np.int64)
    call("tsb_permutation", n, key & M64, out.ctypes.data)
    return out


def epoch_order(samples_per_epoch: int, shuffle_seed: int, epoch: int,
                reshuffle_each_epoch: bool = True) -> np.ndarray:
    """pipeline.py:113-123 (host C++; uploaded to HBM once per epoch by callers)."""
    out = np.empty(samples_per_epoch, dtype=np.int64)
    call("tsb_epoch_order", samples_per_epoch, shuffle_seed & M64, epoch & M64,
         int(bool(reshuffle_each_epoch)), out.ctypes.data)
    return out


def norm_consts(mean=IMAGENET_MEAN, std=IMAGENET_STD) -> tuple[np.ndarray, np.ndarray]:
    """scale = f32(1/(255*std)), bias = f32(-mean/std), rounded once from float64."""
    mean = np.asarray(mean, dtype=np.float64)
    std = np.asarray(std, dtype=np.float64)
    return (1.0 / (255.0 * std)).astype(np.float32), (-mean / std).astype(np.float32)


def _fptr(a):
    if a is None:
        return None
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), a


# -- kernels ------------------------------------------------------------------

def fill_synthetic(out, d_indices, b: int, seed: int, epoch: int, sample_bytes: int,
                   stream=None) -> None:
    """SyntheticSource batch (pipeline.py:183-189) generated in HBM."""
    call("tsb_fill_synthetic", ptr(out), ptr(d_indices), b, seed & M64, epoch & M64,
         sample_bytes, current_stream(stream))


def make_store(out, seed: int, count: int, sample_bytes: int, first: int = 0,
               stream=None) -> None:
    """Materialise a DirectorySource-equivalent store (pipeline.py:139-155)."""
    call("tsb_make_store", ptr(out), seed & M64, first, count, sample_bytes,
         current_stream(stream))


def gather(src, d_indices, b: int, sample_bytes: int, out, stream=None) -> None:
    """Passthrough collate from an HBM or pinned-host store (pipeline.py:190-210)."""
    call("tsb_gather", ptr(src), ptr(d_indices), b, sample_bytes, ptr(out),
         current_stream(stream))


def aug_params(aug_seed: int, epoch: int, d_indices, b: int, pad: int, flip: bool, d_params,
               stream=None) -> None:
    call("tsb_aug_params", aug_seed & M64, epoch & M64, ptr(d_indices), b, pad, int(flip),
         ptr(d_params), current_stream(stream))


def collate_augment(src, d_indices, b: int, h: int, w: int, c: int, pad: int, flip: bool,
                    aug_seed: int, epoch: int, out_kind: int, out, scale=None, bias=None,
                    d_params=None, stream=None) -> None:
    """Fused u8 HWC -> crop/flip -> normalise -> NCHW (SURVEY.md §8a A6')."""
    sc = _fptr(scale)
    bi = _fptr(bias)
    call("tsb_collate_augment", ptr(src), ptr(d_indices), b, h, w, c, pad, int(flip),
         aug_seed & M64, epoch & M64, sc[0] if sc else None, bi[0] if bi else None, out_kind,
         ptr(d_params) or None, ptr(out), current_stream(stream))


def collate_augment_fanout(src, d_indices, b, h, w, c, pad, flip, aug_seed, epoch, out_kind,
                           dsts, scale=None, bias=None, stream=None) -> None:
    sc = _fptr(scale)
    bi = _fptr(bias)
    arr = (ctypes.c_void_p * len(dsts))(*[ptr(d) for d in dsts])
    call("tsb_collate_augment_fanout", ptr(src), ptr(d_indices), b, h, w, c, pad, int(flip),
         aug_seed & M64, epoch & M64, sc[0] if sc else None, bi[0] if bi else None, out_kind,
         arr, len(dsts), current_stream(stream))


def stream_sync(handle: int) -> None:
    """cudaStreamSynchronize on a raw stream handle (no torch objects)."""
    call("tsb_stream_sync", ctypes.c_void_p(handle))


def crc32(data, nbytes: int, d_out, stream=None) -> None:
    """CRC-32/IEEE of device bytes into a device uint32 (wire.py:170-172)."""
    call("tsb_crc32", ptr(data), nbytes, ptr(d_out), None, current_stream(stream))


def fanout(src, dsts, nbytes: int, stream=None) -> None:
    arr = (ctypes.c_void_p * len(dsts))(*[ptr(d) for d in dsts])
    call("tsb_fanout", ptr(src), arr, len(dsts), nbytes, current_stream(stream))


def rebatch_window(slot_ptrs, first: int, count: int, per_slot: int, in_sample_bytes: int,
                   tgt_sample_bytes: int, out, stream=None) -> None:
    """Consumer batch = stream samples [first, first+count) gathered from the
    producer slots it straddles (tsb_rebatch_window)."""
    arr = (ctypes.c_void_p * len(slot_ptrs))(*[int(p) for p in slot_ptrs])
    call("tsb_rebatch_window", arr, len(slot_ptrs), first, count, per_slot, in_sample_bytes,
         tgt_sample_bytes, ptr(out), current_stream(stream))


def rebatch_gather(ring_base, ring_samples: int, sample_bytes: int, first: int, count: int,
                   out, stream=None) -> None:
    call("tsb_rebatch_gather", ptr(ring_base), ring_samples, sample_bytes, first, count,
         ptr(out), current_stream(stream))


__all__ = [
    "OUT_U8", "OUT_F32", "OUT_BF16", "stream_sync", "ptr", "mix64", "derive_key", "permutation",
    "epoch_order", "norm_consts", "fill_synthetic", "make_store", "gather", "aug_params",
    "collate_augment", "collate_augment_fanout", "crc32", "fanout", "rebatch_gather",
    "rebatch_window",
]


def memcpy_async(dst, src, nbytes: int, stream=None) -> None:
    """cudaMemcpyAsync(Default) on the given stream (device/pinned pointers or tensors)."""
    call("tsb_memcpy_async", ptr(dst), ptr(src), nbytes, current_stream(stream))


class DeviceEvent:
    """Raw CUDA event owned by libtsb200 (timing on any stream, incl. inside
    native range calls)."""

    def __init__(self):
        h = ctypes.c_void_p()
        call("tsb_event_create", ctypes.byref(h))
        self.handle = h.value

    @property
    def cuda_event(self) -> int:
        return self.handle

    def record(self, stream=None) -> None:
        call("tsb_event_record", self.handle, current_stream(stream))

    def synchronize(self) -> None:
        call("tsb_event_sync", self.handle)

    def elapsed_ms(self, end: "DeviceEvent") -> float:
        ms = ctypes.c_float()
        call("tsb_event_elapsed_ms", self.handle, end.handle, ctypes.byref(ms))
        return float(ms.value)

    def __del__(self):
        try:
            load().tsb_event_destroy(self.handle)
        except Exception:
            pass


# -- peers (multi-GPU fan-out) -------------------------------------------------

def can_access_peer(dev: int, peer: int) -> bool:
    v = ctypes.c_int(0)
    call("tsb_can_access_peer", dev, peer, ctypes.byref(v))
    return bool(v.value)


def enable_peer(dev: int, peer: int) -> None:
    """Kernels on `dev` may load/store `peer`'s HBM (NVLink P2P); idempotent."""
    call("tsb_enable_peer", dev, peer)
