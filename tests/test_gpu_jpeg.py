"""JPEG source: nvJPEG batched decode in front of the
collate kernel.  The decode itself has no bit-exact oracle (IDCT
implementations differ by a few levels): it is checked against libjpeg
(PIL) within a stated tolerance.  Everything after the decode is bit-exact:
the collate/augment of the decoded pixels equals the oracle's collate of the
same pixels, and the targets are the reference's sample indices."""

import io
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)
Image = pytest.importorskip("PIL.Image")

from paper_2409_18749_b200 import (AugmentSpec, CollateLoader, DatasetSpec,  # noqa: E402
                                   JpegSource)
from paper_2409_18749_b200 import _lib  # noqa: E402
from paper_2409_18749_b200.ring import DeviceRing, produce_range  # noqa: E402

H, W, N, B = 64, 96, 24, 8
DECODE_MAX_ABS, DECODE_MEAN_ABS = 4, 0.6  # vs libjpeg (PIL), 4:4:4 quality 95


def make_jpegs(n=N, h=H, w=W, seed=0):
    rng = np.random.default_rng(seed)
    y, x = np.mgrid[0:h, 0:w].astype(np.float32)
    files, pix = [], []
    for i in range(n):
        f = rng.uniform(0.02, 0.15, 3)
        img = np.stack([127 + 100 * np.sin(f[c] * x + (i + c) * 0.7) * np.cos(f[c] * y * 0.5)
                        for c in range(3)], -1)
        img = np.clip(img + rng.normal(0, 4, img.shape), 0, 255).astype(np.uint8)
        buf = io.BytesIO()
        Image.fromarray(img).save(buf, format="JPEG", quality=95, subsampling=0)
        files.append(buf.getvalue())
        pix.append(np.asarray(Image.open(io.BytesIO(files[-1])).convert("RGB")))
    return files, np.stack(pix)


def available():
    import ctypes

    v = ctypes.c_int(0)
    _lib.call("tsb_jpeg_available", ctypes.byref(v))
    return bool(v.value)


pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not available(), reason="libnvjpeg not present")]


def decode_all(src):
    dec = src.decoder(0, B)
    out = torch.empty(N * H * W * 3, dtype=torch.uint8, device="cuda")
    for k in range(0, N, B):
        dec.decode(np.arange(k, k + B), out[k * H * W * 3:(k + B) * H * W * 3])
    torch.cuda.synchronize()
    return out.cpu().numpy().reshape(N, H, W, 3), dec.backend


def test_decode_matches_libjpeg_within_tolerance():
    files, ref = make_jpegs()
    got, backend = decode_all(JpegSource(files, H, W))
    d = np.abs(got.astype(np.int16) - ref.astype(np.int16))
    print(f"nvJPEG backend={backend} vs libjpeg: max|d|={d.max()} mean|d|={d.mean():.3f}")
    assert d.max() <= DECODE_MAX_ABS and d.mean() <= DECODE_MEAN_ABS


@pytest.mark.parametrize("mode", ["augment_f32", "augment_bf16", "gather"])
def test_jpeg_pipeline_bit_exact_after_decode(oracle, mode):
    files, _ = make_jpegs(seed=1)
    src = JpegSource(files, H, W)
    decoded, _ = decode_all(src)
    store_h = decoded.reshape(-1)
    aug = None if mode == "gather" else AugmentSpec(
        pad=6, flip=True, out_dtype="float32" if mode == "augment_f32" else "bfloat16", seed=4)
    ld = CollateLoader(DatasetSpec(src, N, B, shuffle_seed=2), aug)
    ring = DeviceRing(3, ld.batch_nbytes, 1, control="host")
    ring.set_cursor(0, 0)
    n, L = 6, len(ld)
    got = {}

    def consumer():
        for q in range(1, n + 1):
            s = ring.slot_of(q)
            ring.host_wait_ready(s, q, timeout_s=60)
            got[q] = ring.view(s, (ld.batch_nbytes,), torch.uint8).cpu().numpy().copy()
            ring.host_ack(0, q)

    t = threading.Thread(target=consumer)
    t.start()
    ps = torch.cuda.Stream()
    q = 1
    while q <= n:
        epoch, bi = divmod(q - 1, L)
        m = min(n - q + 1, L - bi)
        a = ld.produce_args(epoch)
        a.gate = _lib.GATE_HOST
        produce_range(ring, a, q, bi, m, [0], stream=ps)
        q += m
    ps.synchronize()
    t.join(60)
    assert not t.is_alive()
    scale, bias = oracle.norm_consts()
    kind = {"augment_f32": 1, "augment_bf16": 2}.get(mode)
    for q in range(1, n + 1):
        epoch, bi = divmod(q - 1, L)
        idx = oracle.epoch_order(N, 2, epoch)[bi * B:(bi + 1) * B]
        if kind is None:
            want = oracle.gather(store_h, idx, H * W * 3)
        else:
            want = oracle.collate_augment(store_h, idx, H, W, 3, 6, True, 4, epoch, kind,
                                          scale, bias)
        assert got[q][:ld.input_nbytes].tobytes() == want.tobytes(), q
        np.testing.assert_array_equal(got[q][ld.input_nbytes:].view(np.int64), idx)
    # the Python-level path (produce_into) agrees with the native one
    buf = torch.empty(ld.batch_nbytes, dtype=torch.uint8, device="cuda")
    ld.produce_into(buf.data_ptr(), 0, 1)
    torch.cuda.synchronize()
    assert buf.cpu().numpy().tobytes() == got[2].tobytes()
    ring.close()
