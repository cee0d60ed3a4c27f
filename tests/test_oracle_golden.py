"""Pin the CPU oracle to golden vectors produced by running the reference.

Mirrors the reference's own known-answer tests
(pkg/tests/test_wire.py:27-46, test_kernels.py:9-63, test_pipeline.py:36-127)
and adds the absolute values the reference tests never froze (SURVEY.md
Appendix A).  CPU only.
"""

import zlib

import numpy as np
import pytest


def test_mix64(golden, oracle):
    for x, want in golden["mix64"]:
        assert oracle.mix64(x) == want
        assert oracle.py_mix64(x) == want
    xs = np.array([x for x, _ in golden["mix64"]], dtype=np.uint64)
    np.testing.assert_array_equal(oracle.np_mix64(xs),
                                  np.array([w for _, w in golden["mix64"]], dtype=np.uint64))


def test_derive_key(golden, oracle):
    for s, e, i, want in golden["derive_key"]:
        assert oracle.derive_key(s, e, i) == want
        assert oracle.py_derive_key(s, e, i) == want


def test_permutation(golden, oracle):
    for case in golden["permutation"]:
        p = oracle.permutation(case["n"], case["key"])
        assert zlib.crc32(p.astype("<i8").tobytes()) == case["crc_i64"]
        assert p[:32].tolist() == case["head"]
        if "perm" in case:
            assert p.tolist() == case["perm"]
        assert sorted(p.tolist()) == list(range(case["n"]))  # bijection (test_kernels.py:33-40)


def test_appendix_a_values(oracle):
    # SURVEY.md Appendix A, produced by the reference
    assert oracle.mix64(1) == 0x5692161D100B05E5
    assert oracle.derive_key(0, 0, 0) == 0x238275BC38FCBE91
    assert oracle.derive_key(0, 0, 0x53485546) == 0x239A8DD44B4BA285
    assert oracle.permutation(10, 42).tolist() == [0, 9, 5, 8, 6, 4, 7, 2, 1, 3]


def test_fill_batch(golden, oracle):
    fb = golden["fill_batch"]
    assert oracle.fill_batch(fb["keys"], fb["wps"]).tolist() == fb["words"]


def test_epoch_order(golden, oracle):
    for case in golden["epoch_order"]:
        o = oracle.epoch_order(case["n"], case["shuffle_seed"], case["epoch"], case["reshuffle"])
        assert zlib.crc32(o.astype("<i8").tobytes()) == case["crc_i64"], case
        assert o[:16].tolist() == case["head"]


@pytest.mark.parametrize("nthreads", [1, 4])
def test_prepare_batch_synthetic(golden, oracle, nthreads):
    for case in golden["prepare_batch"]:
        order = oracle.epoch_order(case["samples_per_epoch"], case["shuffle_seed"], case["epoch"])
        idx = oracle.batch_indices(order, case["batch_index"], case["batch_size"])
        assert idx.tolist() == case["indices"]
        sb = case["nbytes"] // case["batch_size"]
        buf = oracle.prepare_synthetic(case["seed"], case["epoch"], idx, sb, nthreads)
        assert oracle.crc32(buf) == case["crc32"], case["name"]
        assert buf[:8].tolist() == case["head8"]
        assert int(buf.sum(dtype=np.uint64)) == case["sum"]


def test_directory_store_gather(golden, oracle):
    d = golden["directory"]
    store = oracle.make_store(d["seed"], d["num_samples"], d["sample_bytes"])
    sb = d["sample_bytes"]
    for i, want in enumerate(d["file_crc32"]):
        assert oracle.crc32(store[i * sb:(i + 1) * sb]) == want
    for b in d["batches"]:
        order = oracle.epoch_order(d["num_samples"], d["shuffle_seed"], b["epoch"])
        idx = oracle.batch_indices(order, b["batch_index"], d["batch_size"])
        assert idx.tolist() == b["indices"]
        assert oracle.crc32(oracle.gather(store, idx, sb)) == b["crc32"]


def test_rebatch_invariance(golden, oracle):
    r = golden["rebatch"]
    n = r["samples_per_epoch"]
    sb = int(np.prod(r["sample_shape"]))
    for case in r["cases"]:
        order = oracle.epoch_order(n, 0, case["epoch"])
        assert len(order) // case["batch_size"] == case["epoch_len"]
        for j, want in enumerate(case["crc32"]):
            idx = oracle.rebatch_indices(order, case["batch_size"], j)
            assert oracle.crc32(oracle.prepare_synthetic(0, case["epoch"], idx, sb)) == want
    assert r["concat64_eq_512"] is True


def test_crc_known_answers(golden, oracle):
    for hexdata, want in golden["crc32"]:
        data = bytes.fromhex(hexdata)
        assert oracle.crc32(data) == want
        assert oracle.crc32_bitwise(data) == want
    assert oracle.crc32(b"123456789") == 0xCBF43926


def test_crc_combine(oracle):
    rng = np.random.default_rng(1)
    a = rng.integers(0, 256, 1000, dtype=np.uint8).tobytes()
    b = rng.integers(0, 256, 777, dtype=np.uint8).tobytes()
    assert oracle.crc32_combine(oracle.crc32(a), oracle.crc32(b), len(b)) == zlib.crc32(a + b)
    assert oracle.crc32_combine(oracle.crc32(a), oracle.crc32(b""), 0) == zlib.crc32(a)


# -- augment spec: two independent restatements agree (parity unpinned) ----

@pytest.mark.parametrize("out_kind", [0, 1, 2])
@pytest.mark.parametrize("pad,flip", [(16, True), (0, False), (4, True)])
def test_augment_c_vs_numpy(oracle, out_kind, pad, flip):
    h, w, c = 24, 32, 3
    n = 40
    store = oracle.make_store(3, n, h * w * c)
    idx = oracle.epoch_order(n, 0, 1)[:9]
    scale, bias = oracle.norm_consts()
    got = oracle.collate_augment(store, idx, h, w, c, pad, flip, 5, 2, out_kind, scale, bias,
                                 nthreads=2)
    want = oracle.np_collate_augment(store, idx, h, w, c, pad, flip, 5, 2, out_kind, scale, bias)
    np.testing.assert_array_equal(got, want)


def test_aug_params_c_vs_python(oracle):
    idx = np.arange(0, 300, 7)
    np.testing.assert_array_equal(oracle.aug_params(0, 3, idx, 16),
                                  oracle.np_aug_params(0, 3, idx, 16))
    p = oracle.aug_params(0, 0, np.arange(2000), 16)
    assert p[:, :2].min() == 0 and p[:, :2].max() == 32
    assert 0.45 < p[:, 2].mean() < 0.55


def test_augment_explicit_param_table(oracle):
    h, w, c = 8, 16, 3
    store = oracle.make_store(1, 4, h * w * c)
    idx = np.array([2, 0, 3])
    params = np.array([[0, 0, 0], [2, 2, 0], [4, 1, 1]], dtype=np.int32)
    got = oracle.collate_augment(store, idx, h, w, c, 2, True, 0, 0, 0, params=params)
    # identity crop at offset (P, P) without flip reproduces the HWC->CHW transpose
    ident = store[0:h * w * c].reshape(h, w, c).transpose(2, 0, 1)
    np.testing.assert_array_equal(got[1], ident)
    assert (got[0][:, :2, :] == 0).all()  # rows above the image are padding


def test_bf16_rne(oracle):
    x = np.array([1.0, 1.00390625, 1.01171875, -2.5, 3.0e-39, 65504.0], dtype=np.float32)
    import torch

    want = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    np.testing.assert_array_equal(oracle.np_bf16_rne(x), want)
