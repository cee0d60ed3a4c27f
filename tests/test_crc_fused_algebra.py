"""The fused checksum's GF(2) decomposition, restated on the CPU (no GPU).

`csrc/tsb_collate_crc.cuh` never walks the output bytes: each element's
contribution comes from a per-position table of its source byte, runs are
moved to the end of their row, rows to the end of the item segment, and
segments to the end of the slot by constant multiplications, and the target's
raw CRC is XORed in.  This test recomputes exactly that decomposition -- the
same tables (G, the row shift, the per-run segment placement W, the init
term) from the source bytes and the crop params -- for small
batches and checks it against zlib.crc32 of the oracle's collate output plus
the int64 target (the bytes create_segment checksums, bs/payload.py:218).
The GPU tests (tests/test_gpu_crc_fused.py) check the kernel against zlib."""

import zlib

import numpy as np
import pytest

POLY = 0xEDB88320


def multmodp(a: int, b: int) -> int:
    """a(x) * b(x) mod P, reflected (bit 31 = x^0), as zlib's multmodp."""
    m, p = 1 << 31, 0
    while True:
        if a & m:
            p ^= b
            if (a & (m - 1)) == 0:
                break
        m >>= 1
        b = (b >> 1) ^ POLY if b & 1 else b >> 1
    return p


def x8n(n: int) -> int:
    """x^(8n) mod P."""
    p, sq = 1 << 31, 1 << 30
    for _ in range(3):
        sq = multmodp(sq, sq)
    while n:
        if n & 1:
            p = multmodp(sq, p)
        n >>= 1
        sq = multmodp(sq, sq)
    return p


def raw(data: bytes) -> int:
    """Zero-init, no-xorout CRC-32 (linear over GF(2))."""
    return zlib.crc32(data, 0xFFFFFFFF) ^ 0xFFFFFFFF  # zlib starts from ~value


def expand(v: int, k: int) -> int:
    """multmodp(k, v) by bit expansion: bit i of v selects k * e_i (the W tables)."""
    out = 0
    for i in range(32):
        if (v >> i) & 1:
            out ^= multmodp(k, 1 << i)
    return out


@pytest.mark.parametrize("kind,c,b", [(1, 3, 3), (2, 3, 2), (0, 3, 2), (1, 1, 5)])
def test_fused_decomposition_equals_zlib(oracle, kind, c, b):
    h = w = 64          # R = 32: two row blocks; w = 64: two 32-element runs
    pad, aug_seed, epoch, N = 6, 5, 1, 16
    E = {0: 1, 1: 4, 2: 2}[kind]
    store = oracle.make_store(3, N, h * w * c)
    idx = np.array([7, 2, 11, 5, 0][:b], dtype=np.int64)
    scale, bias = oracle.norm_consts()
    out = oracle.collate_augment(store, idx, h, w, c, pad, True, aug_seed, epoch, kind,
                                 scale if kind else None, bias if kind else None)
    slot = out.tobytes() + idx.astype("<i8").tobytes()
    params = oracle.aug_params(aug_seed, epoch, idx, pad)

    # F_c(v): the element bytes the kernel emits for source byte v (from the
    # oracle's own normalisation of every byte value)
    F = []
    for ch in range(c):
        img = np.zeros((1, 1, 256, c), dtype=np.uint8)
        img[0, 0, :, ch] = np.arange(256)
        o = oracle.collate_augment(np.ascontiguousarray(img.reshape(-1)), np.zeros(1, np.int64),
                                   1, 256, c, 0, False, 0, 0, kind,
                                   scale if kind else None, bias if kind else None)
        F.append(o.reshape(c, 256)[ch].tobytes())
    # G_c[v][p] = x^(8 E (31-p)) * raw(F_c(v)): one word per element
    G = [[[multmodp(x8n(E * (31 - p)), raw(F[ch][E * v:E * (v + 1)])) for p in range(32)]
          for v in range(256)] for ch in range(c)]

    R, runs = 32, w // 32
    nrb = h // R
    segb = R * w * E
    tail = 8 * b
    nseg = b * c * nrb
    k_row = [x8n(w * E * (R - 1 - r)) for r in range(R)]
    acc = 0
    src = store.reshape(N, h, w, c)
    for s in range(b):
        oy, ox, fl = (int(t) for t in params[s])
        img = src[idx[s]]
        for ch in range(c):
            for rb in range(nrb):
                seg = (s * c + ch) * nrb + rb
                m = nseg - 1 - seg
                for run in range(runs):
                    x = 0  # the combiner's reduced value for (channel, run) of the segment
                    for r in range(R):
                        y = rb * R + r
                        sy = y + oy - pad
                        part = 0  # raw(row r, run) relative to the run's end
                        for p in range(32):
                            xo = run * 32 + p
                            sx = (w - 1 - xo if fl else xo) + ox - pad
                            v = int(img[sy, sx, ch]) if 0 <= sy < h and 0 <= sx < w else 0
                            part ^= G[ch][v][p]
                        x ^= multmodp(k_row[r], part)  # row r -> the segment's last row
                    # W[run][m]: the run -> the row's end, the segment -> the slot's end
                    acc ^= expand(x, x8n(segb * m + tail + 32 * E * (runs - 1 - run)))
    acc ^= raw(idx.astype("<i8").tobytes())  # the target closes the slot
    init = multmodp(x8n(len(slot)), 0xFFFFFFFF) ^ 0xFFFFFFFF
    assert acc ^ init == zlib.crc32(slot)
