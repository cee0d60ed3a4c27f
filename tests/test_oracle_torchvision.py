"""A third-party pin for the augment spec (SURVEY.md §8a A6'), which has no
reference implementation: the oracle's crop/flip geometry and NCHW layout
are checked bit-exactly against torchvision 0.26's own functional ops on u8
tensors -- ``pad`` (zero fill) -> ``crop(top=oy, left=ox)`` -> ``horizontal_flip``
on the CHW image -- and its normalisation against ``to_dtype(scale=True)`` +
``normalize`` within 1e-6 absolute (torchvision rounds differently: it
divides by 255 and by std; the spec multiplies by 1/(255*std)).
The GPU kernel is pinned to the oracle bit-exactly (tests/test_gpu_*.py), so
this chains the kernel to torchvision."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
tvf = pytest.importorskip("torchvision.transforms.v2.functional")


def _torchvision_u8(sample_hwc, oy, ox, flip, pad, h, w):
    img = torch.from_numpy(sample_hwc).permute(2, 0, 1).contiguous()  # HWC -> CHW
    img = tvf.pad(img, [pad, pad, pad, pad], fill=0)
    img = tvf.crop(img, int(oy), int(ox), h, w)
    if flip:
        img = tvf.horizontal_flip(img)
    return img.numpy()


@pytest.mark.parametrize("h,w,c,pad", [(224, 224, 3, 16), (32, 48, 3, 4), (17, 9, 1, 0),
                                       (40, 24, 3, 7)])
def test_crop_flip_geometry_matches_torchvision(oracle, h, w, c, pad):
    N, B, epoch, aug_seed = 64, 24, 3, 5
    sb = h * w * c
    store = oracle.make_store(7, N, sb)
    idx = oracle.epoch_order(N, 1, epoch)[:B]
    params = oracle.aug_params(aug_seed, epoch, idx, pad)
    got = oracle.collate_augment(store, idx, h, w, c, pad, True, aug_seed, epoch,
                                 oracle.OUT_U8)
    assert got.shape == (B, c, h, w)
    flips = 0
    for s in range(B):
        oy, ox, fl = params[s]
        assert 0 <= oy <= 2 * pad and 0 <= ox <= 2 * pad and fl in (0, 1)
        flips += int(fl)
        sample = store[idx[s] * sb:(idx[s] + 1) * sb].reshape(h, w, c)
        want = _torchvision_u8(sample, oy, ox, fl, pad, h, w)
        np.testing.assert_array_equal(got[s], want, err_msg=f"sample {s} params {params[s]}")
    assert 0 < flips < B  # both branches exercised


def test_normalise_matches_torchvision_within_1e6(oracle):
    h, w, c, pad = 64, 64, 3, 8
    N, B, epoch = 32, 8, 0
    sb = h * w * c
    store = oracle.make_store(0, N, sb)
    idx = np.arange(B, dtype=np.int64)
    params = oracle.aug_params(0, epoch, idx, pad)
    scale, bias = oracle.norm_consts()
    got = oracle.collate_augment(store, idx, h, w, c, pad, True, 0, epoch, oracle.OUT_F32,
                                 scale, bias)
    mean = list(oracle.IMAGENET_MEAN)
    std = list(oracle.IMAGENET_STD)
    worst = 0.0
    for s in range(B):
        u8 = _torchvision_u8(store[idx[s] * sb:(idx[s] + 1) * sb].reshape(h, w, c),
                             *params[s], pad, h, w)
        x = tvf.to_dtype(torch.from_numpy(u8), torch.float32, scale=True)
        want = tvf.normalize(x, mean, std).numpy()
        worst = max(worst, float(np.abs(got[s] - want).max()))
    assert worst <= 1e-6, worst
