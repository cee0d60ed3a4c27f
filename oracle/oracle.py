"""CPU ORACLE for the shared-loading hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` / ``--impl reference`` leg) may import this module, and only
as the checker or the timed CPU baseline.  The product package
``paper_2409_18749_b200`` never imports it; it fails loudly without its CUDA
library instead of falling back here.

Two restatements live here:

* ``lib`` -- ctypes binding of ``ts_oracle.c`` (plain C, OpenMP), which
  restates ``/root/reference/pkg/src/batchsocket/kernels.py:27-140`` and
  ``pipeline.py:25,113-123,139-213`` plus the CRC of ``wire.py:170-172``;
  pinned against golden vectors produced by running the reference itself
  (``tests/golden/make_golden.py`` -> ``tests/golden/golden.json``).
* pure numpy functions (``np_*``) -- an independent restatement, used to
  cross-check the C code, including the NEW augment spec (SURVEY.md §8a
  A6').  The augment has no reference implementation: its parity is
  "unpinned" (pinned only by the agreement of these two restatements).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libts_oracle.so")

GAMMA = 0x9E3779B97F4A7C15
MIX1 = 0xBF58476D1CE4E5B9
MIX2 = 0x94D049BB133111EB
M64 = (1 << 64) - 1
SHUFFLE_DOMAIN = 0x53485546  # pipeline.py:25
AUG_DOMAIN = 0x41554731  # "AUG1"

IMAGENET_MEAN = (0.485, 0.456, 0.406)
IMAGENET_STD = (0.229, 0.224, 0.225)

OUT_U8, OUT_F32, OUT_BF16 = 0, 1, 2


def build() -> str:
    """Compile ts_oracle.c -> libts_oracle.so (make; gcc + OpenMP)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


_lib = None


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        build()
    L = ctypes.CDLL(LIB_PATH)
    u64, i64, i32, vp = ctypes.c_uint64, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
    L.tso_mix64.restype = u64
    L.tso_mix64.argtypes = [u64]
    L.tso_derive_key.restype = u64
    L.tso_derive_key.argtypes = [u64, u64, u64]
    L.tso_permutation.argtypes = [i64, u64, vp]
    L.tso_epoch_order.argtypes = [i64, u64, u64, i32, vp]
    L.tso_fill_batch.argtypes = [vp, vp, i64, i64]
    L.tso_prepare_synthetic.argtypes = [u64, u64, vp, i64, i64, vp, i32]
    L.tso_make_store.argtypes = [u64, i64, i64, i64, vp, i32]
    L.tso_gather.argtypes = [vp, vp, i64, i64, vp, i32]
    L.tso_aug_params.argtypes = [u64, u64, vp, i64, i32, i32, vp]
    L.tso_norm_consts.argtypes = [vp, vp, i32, vp, vp]
    L.tso_collate_augment.argtypes = [vp, vp, i64, i32, i32, i32, i32, i32, u64, u64,
                                      vp, vp, i32, vp, vp, i32]
    L.tso_crc32.restype = ctypes.c_uint32
    L.tso_crc32.argtypes = [vp, ctypes.c_size_t, ctypes.c_uint32]
    L.tso_crc32_bitwise.restype = ctypes.c_uint32
    L.tso_crc32_bitwise.argtypes = [vp, ctypes.c_size_t]
    L.tso_crc32_combine.restype = ctypes.c_uint32
    L.tso_crc32_combine.argtypes = [ctypes.c_uint32, ctypes.c_uint32, u64]
    L.tso_num_threads.restype = i32
    _lib = L
    return L


def _p(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


def nthreads_default() -> int:
    return load().tso_num_threads()


# -- C oracle wrappers -------------------------------------------------------

def mix64(x: int) -> int:
    return int(load().tso_mix64(x & M64))


def derive_key(seed: int, epoch: int, index: int) -> int:
    return int(load().tso_derive_key(seed & M64, epoch & M64, index & M64))


def permutation(n: int, key: int) -> np.ndarray:
    out = np.empty(n, dtype=np.int64)
    if n:
        load().tso_permutation(n, key & M64, _p(out))
    return out


def epoch_order(samples_per_epoch: int, shuffle_seed: int, epoch: int,
                reshuffle_each_epoch: bool = True) -> np.ndarray:
    out = np.empty(samples_per_epoch, dtype=np.int64)
    load().tso_epoch_order(samples_per_epoch, shuffle_seed & M64, epoch & M64,
                           int(bool(reshuffle_each_epoch)), _p(out))
    return out


def fill_batch(keys, words_per_sample: int) -> np.ndarray:
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    out = np.empty(len(keys) * words_per_sample, dtype=np.uint64)
    load().tso_fill_batch(_p(out), _p(keys), len(keys), words_per_sample)
    return out


def batch_indices(order: np.ndarray, batch_index: int, batch_size: int) -> np.ndarray:
    """pipeline.py:178-180 (drop-last handled by the caller's epoch_len)."""
    lo = batch_index * batch_size
    return np.ascontiguousarray(order[lo:lo + batch_size])


def prepare_synthetic(seed: int, epoch: int, indices: np.ndarray, sample_bytes: int,
                      nthreads: int = 1) -> np.ndarray:
    indices = np.ascontiguousarray(indices, dtype=np.int64)
    out = np.empty(len(indices) * sample_bytes, dtype=np.uint8)
    load().tso_prepare_synthetic(seed & M64, epoch & M64, _p(indices), len(indices),
                                 sample_bytes, _p(out), nthreads)
    return out


def make_store(seed: int, count: int, sample_bytes: int, first: int = 0,
               nthreads: int = 0) -> np.ndarray:
    out = np.empty(count * sample_bytes, dtype=np.uint8)
    load().tso_make_store(seed & M64, first, count, sample_bytes, _p(out),
                          nthreads or nthreads_default())
    return out


def gather(store: np.ndarray, indices: np.ndarray, sample_bytes: int,
           nthreads: int = 1, out: np.ndarray | None = None) -> np.ndarray:
    indices = np.ascontiguousarray(indices, dtype=np.int64)
    if out is None:
        out = np.empty(len(indices) * sample_bytes, dtype=np.uint8)
    load().tso_gather(_p(store), _p(indices), len(indices), sample_bytes, _p(out), nthreads)
    return out


def aug_params(aug_seed: int, epoch: int, indices: np.ndarray, pad: int,
               flip: bool = True) -> np.ndarray:
    indices = np.ascontiguousarray(indices, dtype=np.int64)
    out = np.empty((len(indices), 3), dtype=np.int32)
    load().tso_aug_params(aug_seed & M64, epoch & M64, _p(indices), len(indices), pad,
                          int(flip), _p(out))
    return out


def norm_consts(mean=IMAGENET_MEAN, std=IMAGENET_STD):
    mean = np.ascontiguousarray(mean, dtype=np.float64)
    std = np.ascontiguousarray(std, dtype=np.float64)
    scale = np.empty(len(mean), dtype=np.float32)
    bias = np.empty(len(mean), dtype=np.float32)
    load().tso_norm_consts(_p(mean), _p(std), len(mean), _p(scale), _p(bias))
    return scale, bias


def collate_augment(store: np.ndarray, indices: np.ndarray, h: int, w: int, c: int,
                    pad: int, flip: bool, aug_seed: int, epoch: int, out_kind: int,
                    scale=None, bias=None, params=None, nthreads: int = 1,
                    out: np.ndarray | None = None) -> np.ndarray:
    indices = np.ascontiguousarray(indices, dtype=np.int64)
    b = len(indices)
    dt = {OUT_U8: np.uint8, OUT_F32: np.float32, OUT_BF16: np.uint16}[out_kind]
    if out is None:
        out = np.empty((b, c, h, w), dtype=dt)
    sc = None if scale is None else np.ascontiguousarray(scale, dtype=np.float32)
    bi = None if bias is None else np.ascontiguousarray(bias, dtype=np.float32)
    pr = None if params is None else np.ascontiguousarray(params, dtype=np.int32)
    load().tso_collate_augment(_p(store), _p(indices), b, h, w, c, pad, int(flip),
                               aug_seed & M64, epoch & M64, _p(sc), _p(bi), out_kind,
                               _p(pr), _p(out), nthreads)
    return out


def crc32(data, prev: int = 0) -> int:
    a = np.frombuffer(memoryview(data).cast("B"), dtype=np.uint8) if not isinstance(
        data, np.ndarray) else data.reshape(-1).view(np.uint8)
    a = np.ascontiguousarray(a)
    return int(load().tso_crc32(_p(a), a.nbytes, prev & 0xFFFFFFFF))


def crc32_bitwise(data: bytes) -> int:
    a = np.frombuffer(data, dtype=np.uint8)
    return int(load().tso_crc32_bitwise(_p(a), a.nbytes))


def crc32_combine(crc1: int, crc2: int, len2: int) -> int:
    return int(load().tso_crc32_combine(crc1, crc2, len2))


def rebatch_indices(order: np.ndarray, batch_size: int, batch_index: int) -> np.ndarray:
    """Consumer with its own batch size: order[j*b:(j+1)*b], j < N // b."""
    if batch_index >= len(order) // batch_size:
        raise ValueError("batch_index beyond drop-last epoch_len")
    return batch_indices(order, batch_index, batch_size)


# -- independent numpy restatement (cross-check of the C code) -------------

_U = np.uint64


def np_mix64(z: np.ndarray) -> np.ndarray:
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> _U(30))) * _U(MIX1)
        z = (z ^ (z >> _U(27))) * _U(MIX2)
    return z ^ (z >> _U(31))


def py_mix64(x: int) -> int:
    z = x & M64
    z = ((z ^ (z >> 30)) * MIX1) & M64
    z = ((z ^ (z >> 27)) * MIX2) & M64
    return z ^ (z >> 31)


def py_derive_key(seed: int, epoch: int, index: int) -> int:
    h = py_mix64((seed + GAMMA) & M64)
    h = py_mix64(((h ^ epoch) + GAMMA) & M64)
    h = py_mix64(((h ^ index) + GAMMA) & M64)
    return h


def np_aug_params(aug_seed: int, epoch: int, indices, pad: int, flip: bool = True):
    s = py_mix64((aug_seed ^ AUG_DOMAIN) & M64)
    out = np.empty((len(indices), 3), dtype=np.int32)
    m = 2 * pad + 1
    for i, idx in enumerate(indices):
        ka = py_derive_key(s, epoch, int(idx))
        out[i, 0] = py_mix64((ka + GAMMA) & M64) % m
        out[i, 1] = py_mix64((ka + 2 * GAMMA) & M64) % m
        out[i, 2] = (py_mix64((ka + 3 * GAMMA) & M64) & 1) if flip else 0
    return out


def np_bf16_rne(x: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = (u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    return r.astype(np.uint16)


def np_collate_augment(store: np.ndarray, indices, h, w, c, pad, flip, aug_seed, epoch,
                       out_kind, scale=None, bias=None):
    """Vectorised numpy version of the augment spec (pad -> crop -> flip -> normalise)."""
    params = np_aug_params(aug_seed, epoch, indices, pad, flip)
    sb = h * w * c
    outs = []
    for i, idx in enumerate(indices):
        img = store[int(idx) * sb:(int(idx) + 1) * sb].reshape(h, w, c)
        padded = np.zeros((h + 2 * pad, w + 2 * pad, c), dtype=np.uint8)
        padded[pad:pad + h, pad:pad + w] = img
        oy, ox, fl = (int(v) for v in params[i])
        crop = padded[oy:oy + h, ox:ox + w]
        if fl:
            crop = crop[:, ::-1]
        chw = np.ascontiguousarray(crop.transpose(2, 0, 1))
        if out_kind == OUT_U8:
            outs.append(chw)
            continue
        sc = np.asarray(scale, dtype=np.float32).reshape(c, 1, 1)
        bi = np.asarray(bias, dtype=np.float32).reshape(c, 1, 1)
        v = chw.astype(np.float32) * sc + bi  # float32 ops, two roundings
        outs.append(v.astype(np.float32) if out_kind == OUT_F32 else np_bf16_rne(v))
    return np.stack(outs)
