"""GPU parity of the sm_100a kernels against the CPU oracle / golden vectors.

Every test goes through the C ABI (libtsb200.so via ctypes).  Bars
(BASELINE.json north_star): indices, ordering and u8 payloads bit-exact;
fp32 within 1e-6 relative (the kernel is in fact bit-exact: no FMA, same
two roundings as the oracle); bf16 within 1 ulp (in fact bit-exact RNE).
"""

import zlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU host
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2409_18749_b200 import dataplane as dp  # noqa: E402
from paper_2409_18749_b200.ring import DeviceRing, sync_mode  # noqa: E402

FP32_RTOL = 1e-6  # north_star tolerance (the kernel is bit-exact)
BF16_ULP = 1


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host_bytes(t) -> bytes:
    torch.cuda.synchronize()
    return t.cpu().numpy().tobytes()


def test_library_arch():
    info = torch.cuda.get_device_capability()
    assert info[0] == 10, f"expected sm_100 (B200), got {info}"


def test_epoch_order_host_native(golden, oracle):
    for case in golden["epoch_order"]:
        o = dp.epoch_order(case["n"], case["shuffle_seed"], case["epoch"], case["reshuffle"])
        assert zlib.crc32(o.astype("<i8").tobytes()) == case["crc_i64"]


@pytest.mark.parametrize("case_i", range(12))
def test_fill_synthetic_matches_reference(golden, case_i):
    case = golden["prepare_batch"][case_i]
    idx = dev(np.array(case["indices"], dtype=np.int64))
    sb = case["nbytes"] // case["batch_size"]
    out = torch.empty(case["nbytes"], dtype=torch.uint8, device="cuda")
    dp.fill_synthetic(out, idx, case["batch_size"], case["seed"], case["epoch"], sb)
    data = host_bytes(out)
    assert zlib.crc32(data) == case["crc32"], case["name"]
    assert list(data[:8]) == case["head8"]
    # device CRC of the same slot equals the reference checksum
    crc = torch.zeros(1, dtype=torch.int32, device="cuda")
    dp.crc32(out, case["nbytes"], crc)
    torch.cuda.synchronize()
    assert int(crc.item()) & 0xFFFFFFFF == case["crc32"]


def test_store_gather_matches_directory_source(golden):
    d = golden["directory"]
    sb = d["sample_bytes"]
    store = torch.empty(d["num_samples"] * sb, dtype=torch.uint8, device="cuda")
    dp.make_store(store, d["seed"], d["num_samples"], sb)
    s = store.cpu().numpy()
    for i, want in enumerate(d["file_crc32"]):
        assert zlib.crc32(s[i * sb:(i + 1) * sb].tobytes()) == want
    out = torch.empty(d["batch_size"] * sb, dtype=torch.uint8, device="cuda")
    for b in d["batches"]:
        dp.gather(store, dev(np.array(b["indices"], dtype=np.int64)), d["batch_size"], sb, out)
        assert zlib.crc32(host_bytes(out)) == b["crc32"]


def test_gather_from_pinned_host_store(golden, oracle):
    """Ingest straight from pinned host memory (device-mapped) -- the e2e source."""
    d = golden["directory"]
    sb = d["sample_bytes"]
    host = torch.from_numpy(oracle.make_store(d["seed"], d["num_samples"], sb)).pin_memory()
    out = torch.empty(d["batch_size"] * sb, dtype=torch.uint8, device="cuda")
    for b in d["batches"]:
        dp.gather(host, dev(np.array(b["indices"], dtype=np.int64)), d["batch_size"], sb, out)
        assert zlib.crc32(host_bytes(out)) == b["crc32"]


@pytest.mark.parametrize("sb", [8, 24, 4104, 150528])
def test_gather_odd_sizes(oracle, sb):
    n, b = 37, 11
    store = oracle.make_store(2, n, sb)
    idx = oracle.epoch_order(n, 1, 0)[:b]
    out = torch.empty(b * sb, dtype=torch.uint8, device="cuda")
    dp.gather(dev(store), dev(idx), b, sb, out)
    assert host_bytes(out) == oracle.gather(store, idx, sb).tobytes()


AUG_CASES = [
    # h, w, c, pad, flip, b
    (224, 224, 3, 16, True, 16),
    (224, 224, 3, 0, False, 4),
    (32, 32, 3, 4, True, 33),
    (17, 48, 3, 8, True, 5),   # h not a multiple of the row block
    (64, 64, 1, 2, True, 7),
]


@pytest.mark.parametrize("out_kind", [0, 1, 2])
@pytest.mark.parametrize("h,w,c,pad,flip,b", AUG_CASES)
def test_collate_augment_parity(oracle, out_kind, h, w, c, pad, flip, b):
    if w % {0: 16, 1: 4, 2: 8}[out_kind]:
        pytest.skip("width not vectorisable for this output kind")
    n = max(64, b)
    store = oracle.make_store(7, n, h * w * c)
    idx = oracle.epoch_order(n, 0, 3)[:b]
    mean = (0.485, 0.456, 0.406, 0.5)[:c]
    std = (0.229, 0.224, 0.225, 0.25)[:c]
    scale, bias = oracle.norm_consts(mean, std)
    np.testing.assert_array_equal(scale, dp.norm_consts(mean, std)[0])
    want = oracle.collate_augment(store, idx, h, w, c, pad, flip, 11, 3, out_kind, scale, bias,
                                  nthreads=4)
    tdt = {0: torch.uint8, 1: torch.float32, 2: torch.int16}[out_kind]
    out = torch.empty((b, c, h, w), dtype=tdt, device="cuda")
    dp.collate_augment(dev(store), dev(idx), b, h, w, c, pad, flip, 11, 3, out_kind, out,
                       scale=scale, bias=bias)
    got = out.cpu().numpy()
    if out_kind == 1:
        np.testing.assert_allclose(got, want, rtol=FP32_RTOL, atol=0)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), "expected bit-exact"
    elif out_kind == 2:
        g = got.view(np.uint16).astype(np.int64)
        w_ = want.view(np.uint16).astype(np.int64)
        assert np.abs(g - w_).max() <= BF16_ULP
        assert np.array_equal(g, w_), "expected bit-exact RNE"
    else:
        np.testing.assert_array_equal(got, want)


def test_collate_param_table_and_pinned_source(oracle):
    h, w, c, b, n, pad = 224, 224, 3, 8, 40, 16
    store = oracle.make_store(1, n, h * w * c)
    idx = oracle.epoch_order(n, 2, 1)[:b]
    scale, bias = oracle.norm_consts()
    want = oracle.collate_augment(store, idx, h, w, c, pad, True, 0, 1, 2, scale, bias)
    params = torch.empty((b, 3), dtype=torch.int32, device="cuda")
    didx = dev(idx)
    dp.aug_params(0, 1, didx, b, pad, True, params)
    np.testing.assert_array_equal(params.cpu().numpy(), oracle.aug_params(0, 1, idx, pad))
    pinned = torch.from_numpy(store).pin_memory()
    out = torch.empty((b, c, h, w), dtype=torch.int16, device="cuda")
    dp.collate_augment(pinned, didx, b, h, w, c, pad, True, 0, 1, 2, out, scale, bias,
                       d_params=params)
    np.testing.assert_array_equal(out.cpu().numpy().view(np.uint16), want)


@pytest.mark.parametrize("n", [0, 1, 3, 63, 64, 2047, 2048, 2049, 65536 + 5, 3 * 2**20 + 17])
@pytest.mark.parametrize("offset", [0, 1, 16])
def test_crc32_device(n, offset):
    rng = np.random.default_rng(n + offset)
    data = rng.integers(0, 256, n + offset, dtype=np.uint8)
    t = dev(data)
    out = torch.zeros(1, dtype=torch.int32, device="cuda")
    dp.crc32(t.data_ptr() + offset, n, out)
    torch.cuda.synchronize()
    assert int(out.item()) & 0xFFFFFFFF == zlib.crc32(data[offset:].tobytes())


@pytest.mark.parametrize("n", [4608 * 64, 4608 * 64 + 16, 4608 * 1000 + 16, 4608 * 777 + 4592,
                               4608 * 5000 - 48, 154142720])
@pytest.mark.parametrize("offset", [0, 16, 48])
def test_crc32_tile_kernel_sizes(n, offset):
    """The TMA tile CRC kernel (16 B-aligned buffers of >= 64 tiles): exact
    multiples of the 4,608-byte tile, a front-padded first tile (z = 16 ..
    4,592 virtual zeros), many warps' runs, and a whole f32 C2 batch."""
    rng = np.random.default_rng(n % 9973 + offset)
    data = rng.integers(0, 256, n + offset, dtype=np.uint8)
    t = dev(data)
    out = torch.zeros(1, dtype=torch.int32, device="cuda")
    dp.crc32(t.data_ptr() + offset, n, out)
    torch.cuda.synchronize()
    assert int(out.item()) & 0xFFFFFFFF == zlib.crc32(data[offset:].tobytes())


def test_crc32_known_answers(golden):
    out = torch.zeros(1, dtype=torch.int32, device="cuda")
    for hexdata, want in golden["crc32"]:
        data = bytes.fromhex(hexdata)
        t = dev(np.frombuffer(data, dtype=np.uint8).copy()) if data else torch.zeros(
            1, dtype=torch.uint8, device="cuda")
        dp.crc32(t, len(data), out)
        torch.cuda.synchronize()
        assert int(out.item()) & 0xFFFFFFFF == want


def test_fanout_and_fused_collate_fanout(oracle):
    nbytes = 3 * 2**20 + 48
    src = dev(np.random.default_rng(0).integers(0, 256, nbytes, dtype=np.uint8))
    dsts = [torch.zeros(nbytes, dtype=torch.uint8, device="cuda") for _ in range(3)]
    dp.fanout(src, dsts, nbytes)
    torch.cuda.synchronize()
    for d in dsts:
        assert torch.equal(d, src)
    h, w, c, b = 64, 64, 3, 6
    store = oracle.make_store(4, 20, h * w * c)
    idx = oracle.epoch_order(20, 0, 0)[:b]
    scale, bias = oracle.norm_consts()
    want = oracle.collate_augment(store, idx, h, w, c, 4, True, 9, 2, 1, scale, bias)
    outs = [torch.empty((b, c, h, w), dtype=torch.float32, device="cuda") for _ in range(4)]
    dp.collate_augment_fanout(dev(store), dev(idx), b, h, w, c, 4, True, 9, 2, 1, outs,
                              scale=scale, bias=bias)
    for o in outs:
        np.testing.assert_array_equal(o.cpu().numpy(), want)


def test_rebatch_gather_wraps(oracle):
    ring_samples, sb = 10, 4104
    ring = dev(oracle.make_store(3, ring_samples, sb))
    host = ring.cpu().numpy()
    out = torch.empty(7 * sb, dtype=torch.uint8, device="cuda")
    dp.rebatch_gather(ring, ring_samples, sb, 6, 7, out)
    want = np.concatenate([host[((6 + j) % ring_samples) * sb:((6 + j) % ring_samples + 1) * sb]
                           for j in range(7)])
    assert host_bytes(out) == want.tobytes()


def test_ring_device_sync_in_process():
    ring = DeviceRing(slots=4, slot_bytes=1 << 20, max_consumers=4)
    prod = torch.cuda.Stream()
    cons = [torch.cuda.Stream() for _ in range(2)]
    src = torch.arange(1 << 18, dtype=torch.int32, device="cuda")
    for seq in range(1, 13):
        slot = ring.slot_of(seq)
        with torch.cuda.stream(prod):
            ring.wait_free([0, 1], seq - ring.slots, prod)
            v = ring.view(slot, (1 << 18,), torch.int32)
            v.copy_(src + seq)
            ring.publish(slot, seq, prod)
        for k, s in enumerate(cons):
            with torch.cuda.stream(s):
                ring.wait_ready(slot, seq, s)
                got = ring.view(slot, (1 << 18,), torch.int32)
                assert_t = (got - seq).eq(src).all()
                ring.ack(k, seq, s)
                s.synchronize()
                assert bool(assert_t.item())
    torch.cuda.synchronize()
    assert ring.read_cursor(0) == 12 and ring.read_cursor(1) == 12
    assert ring.read_ready(ring.slot_of(12)) == 12
    ring.evict(1)
    assert ring.read_cursor(1) == 1 << 62
    print("sync mode:", sync_mode())
    ring.close()


def test_zero_copy_view_is_the_slot():
    ring = DeviceRing(slots=2, slot_bytes=4096, max_consumers=1)
    a = ring.view(1, (1024,), torch.float32)
    a.fill_(3.5)
    b = ring.view(1, (2048,), torch.bfloat16)
    assert a.data_ptr() == b.data_ptr() == ring.slot_ptr(1)
    torch.cuda.synchronize()
    assert float(a.sum()) == 3.5 * 1024


def test_directory_source_files_and_batches_match_reference(golden, tmp_path):
    """StoreSource.write_directory / from_directory (pipeline.py:45-54,139-155,
    190-210): the files equal the reference's write_directory_dataset bytes
    and the gathered batches equal its prepare_batch (golden CRCs)."""
    import zlib

    from paper_2409_18749_b200 import CollateLoader, DatasetSpec, StoreSource

    d = golden["directory"]
    StoreSource.write_directory(str(tmp_path), d["num_samples"], d["sample_bytes"], d["seed"])
    for i, want in enumerate(d["file_crc32"]):
        data = (tmp_path / f"sample-{i:08d}.bin").read_bytes()
        assert zlib.crc32(data) == want
    for location in ("pinned", "hbm"):
        store = StoreSource.from_directory(str(tmp_path), (d["sample_bytes"],),
                                           location=location)
        ld = CollateLoader(DatasetSpec(store, d["num_samples"], d["batch_size"],
                                       shuffle_seed=d["shuffle_seed"]))
        for case in d["batches"]:
            buf = torch.empty(ld.batch_nbytes, dtype=torch.uint8, device="cuda")
            ld.produce_into(buf.data_ptr(), case["epoch"], case["batch_index"])
            got = buf.cpu().numpy()
            assert zlib.crc32(got[:ld.input_nbytes].tobytes()) == case["crc32"]
            np.testing.assert_array_equal(got[ld.input_nbytes:].view(np.int64), case["indices"])
    (tmp_path / "sample-00000003.bin").write_bytes(b"short")
    with pytest.raises(ValueError, match="expected"):
        StoreSource.from_directory(str(tmp_path), (d["sample_bytes"],))


@pytest.mark.parametrize("mean,std", [
    ((0.485, 0.456, 0.406), (0.229, 0.224, 0.225)),        # one-FMA bf16 path is exact here
    ((0.8041, 0.7499, 0.6343), (0.4834, 0.4703, 0.3993)),  # ... and not here (channel 0)
])
def test_bf16_fma_path_selection_is_bit_exact(oracle, mean, std):
    """The bf16 kernel takes one FFMA2 per pair only when, for the batch's
    scale/bias, the single rounding gives the oracle's bf16 for all 256 byte
    values of every channel (checked on the host); otherwise it keeps the two
    roundings.  Either way the output is the oracle's, bit for bit."""
    h, w, c, b, pad = 32, 64, 3, 16, 4
    store = oracle.make_store(3, 64, h * w * c)
    idx = oracle.epoch_order(64, 0, 1)[:b]
    scale, bias = oracle.norm_consts(mean, std)
    u = np.arange(256, dtype=np.float32)
    two = ((u[:, None] * scale).astype(np.float32) + bias).astype(np.float32)
    fma = (u[:, None].astype(np.float64) * scale.astype(np.float64) + bias).astype(np.float32)

    def rne(x):
        bits = x.view(np.uint32).astype(np.uint64)
        return (bits + 0x7FFF + ((bits >> 16) & 1)) >> 16

    exact_fma = np.array_equal(rne(two), rne(fma))
    assert exact_fma == (mean[0] == 0.485)  # the two cases really differ
    want = oracle.collate_augment(store, idx, h, w, c, pad, True, 5, 1, 2, scale, bias)
    out = torch.empty((b, c, h, w), dtype=torch.int16, device="cuda")
    dp.collate_augment(dev(store), dev(idx), b, h, w, c, pad, True, 5, 1, 2, out,
                       scale=scale, bias=bias)
    np.testing.assert_array_equal(out.cpu().numpy().view(np.uint16), want)
