"""BASELINE.json's configs at their real sizes through the public API.

* C3's output: a whole B=256 224x224x3 -> bf16 NCHW batch (and the u8
  crop/flip-only output) bit-exact against the oracle.
* C4: ``TensorProducer`` over B=512 bf16 slots with ``SharedLoader(batch_size=b)``
  consumers for b in {64, 128, 256, 512} plus b=384, whose windows straddle
  slots and so run the rebatch gather kernel at size.  Each consumer batch j
  must be the reference's batch for b: samples ``order[j*b:(j+1)*b]``
  (bs/pipeline.py:77-79,113-123), checked by device CRC against the oracle's
  CRC of the same collate.
* C5: video (16,3,112,112) u8 B=16 and LLM (2048,) int32 B=256 through
  ``TensorProducer`` to 8 consumers: every consumer's batches equal the
  reference's ``prepare_batch`` -- the CRCs frozen by running the reference
  (tests/golden) and the oracle's CRC of every other batch.

Consumers run as threads of this process, each on its own CUDA stream (one
process per consumer behaves the same way, tests/test_gpu_facade.py)."""

import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2409_18749_b200 import (AugmentSpec, CollateLoader, DatasetSpec,  # noqa: E402
                                   SharedLoader, StoreSource, SyntheticSource, TensorProducer)
from paper_2409_18749_b200 import dataplane as dp  # noqa: E402
from paper_2409_18749_b200._lib import GATE_HOST  # noqa: E402
from paper_2409_18749_b200.ring import DeviceRing, produce_range  # noqa: E402
from paper_2409_18749_b200.wire import DType  # noqa: E402

H, W, C, PAD = 224, 224, 3, 16
SB = H * W * C


def _oracle_batch(oracle, epoch, idx, kind, seed=0, aug_seed=0, nthreads=8):
    """Oracle collate+augment of store samples `idx` (store sample i =
    fill(derive_key(seed, 0, i)), pipeline.py:139-155) -- only those samples
    are materialised."""
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    mini = oracle.prepare_synthetic(seed, 0, idx, SB, nthreads)
    params = oracle.aug_params(aug_seed, epoch, idx, PAD)
    scale, bias = oracle.norm_consts()
    return oracle.collate_augment(mini, np.arange(len(idx), dtype=np.int64), H, W, C, PAD, True,
                                  aug_seed, epoch, kind, scale if kind else None,
                                  bias if kind else None, params=params, nthreads=nthreads)


@pytest.mark.parametrize("out_dtype,kind", [("bfloat16", 2), ("uint8", 0)])
def test_full_b256_batch_bit_exact(oracle, out_dtype, kind):
    """C3's dtype at its full batch: 256 x 3 x 224 x 224 bf16 (77 MB) through
    the native producer loop, bit-exact; the u8 output is the crop/flip alone."""
    N, B = 16384, 256
    ld = CollateLoader(DatasetSpec(StoreSource.synthetic(0, N, (H, W, C)), N, B),
                       AugmentSpec(pad=PAD, flip=True, out_dtype=out_dtype))
    ring = DeviceRing(2, ld.batch_nbytes, 1, control="host")
    a = ld.produce_args(1)
    a.gate = GATE_HOST
    produce_range(ring, a, 1, 5, 1, [])
    torch.cuda.synchronize()
    got = ring.view(0, (ld.batch_nbytes,), torch.uint8).cpu().numpy()
    idx = oracle.epoch_order(N, 0, 1)[5 * B:6 * B]
    want = _oracle_batch(oracle, 1, idx, kind)
    assert got[:ld.input_nbytes].tobytes() == want.tobytes()
    np.testing.assert_array_equal(got[ld.input_nbytes:].view(np.int64), idx)
    ring.close()


def _run_facade(endpoints, ld, consumer_kws, epochs, record, **pkw):
    b, a = endpoints
    producer = TensorProducer(ld, broadcast=b, aggregate=a, heartbeat_timeout_s=30.0,
                              min_consumers=len(consumer_kws), **pkw)

    def run():
        for _ in range(epochs):
            for _ in producer:
                pass
        producer.join(60)

    pt = threading.Thread(target=run, daemon=True)
    pt.start()
    outs = [[] for _ in consumer_kws]
    errs = []

    def consume(i, kw):
        loader = SharedLoader(b, a, consumer_id=200 + i, **kw)
        crc = None
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for e in range(epochs):
                    for inp, tgt in loader:
                        if crc is None:
                            crc = torch.zeros(1, dtype=torch.int32, device="cuda")
                        outs[i].append(record(e, inp, tgt, crc, s))
                    if loader.finished:
                        break
        except Exception:  # noqa: BLE001
            import traceback

            errs.append(traceback.format_exc())
        finally:
            loader.close()

    ts = [threading.Thread(target=consume, args=(i, kw)) for i, kw in enumerate(consumer_kws)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(600)
        assert not t.is_alive(), "consumer hung"
    pt.join(120)
    assert not errs, errs[0]
    return producer, outs


def _device_crc(inp, crc, stream) -> int:
    """CRC-32 of a consumer's (contiguous) view, on the device."""
    nbytes = inp.numel() * inp.element_size()
    dp.crc32(inp.data_ptr(), nbytes, crc, stream)
    stream.synchronize()
    return int(crc.item()) & 0xFFFFFFFF


def test_c4_heterogeneous_consumers_full_size(tmp_path, oracle):
    """C4 at its real batch sizes: B=512 bf16 producer slots (154 MB), one
    consumer per b in {64, 128, 256, 512, 384}.  384 straddles slots, so the
    rebatch gather kernel runs on 115 MB windows; the others are zero-copy
    windows.  Every consumer batch equals the oracle's collate of
    order[j*b:(j+1)*b], N // b batches per epoch."""
    N, P = 4096, 512
    sizes = [64, 128, 256, 512, 384]
    ld = CollateLoader(DatasetSpec(StoreSource.synthetic(0, N, (H, W, C)), N, P),
                       AugmentSpec(pad=PAD, flip=True, out_dtype="bfloat16"))

    def record(e, inp, tgt, crc, s):
        assert inp.is_contiguous() and inp.dtype == torch.bfloat16
        return e, inp.shape[0], _device_crc(inp, crc, s), tgt.cpu().numpy().copy()

    eps = (f"unix:{tmp_path}/c4b.sock", f"unix:{tmp_path}/c4a.sock")
    producer, outs = _run_facade(eps, ld, [{"batch_size": b} for b in sizes], 1, record,
                                 ring_slots=4)
    order = oracle.epoch_order(N, 0, 0)
    cache = {}
    for b, got in zip(sizes, outs):
        assert len(got) == N // b, (b, len(got))
        for j, (e, n, crc, tgt) in enumerate(got):
            idx = order[j * b:(j + 1) * b]
            assert e == 0 and n == b
            np.testing.assert_array_equal(tgt, idx, err_msg=f"b={b} batch {j}")
            key = (j * b, b)
            if key not in cache:
                cache[key] = oracle.crc32(_oracle_batch(oracle, 0, idx, 2))
            assert crc == cache[key], f"b={b} batch {j}: {crc:#x} != {cache[key]:#x}"
    producer.close()


@pytest.mark.parametrize("case_i,epochs", [(8, 4), (6, 2)])  # video B=16; LLM B=256
def test_c5_eight_consumers_match_reference(tmp_path, golden, oracle, case_i, epochs):
    """C5 through the facade: 8 consumers each receive every batch, equal to
    the reference's prepare_batch (golden CRCs where frozen, the oracle's
    synthetic fill of the same indices everywhere else)."""
    case = golden["prepare_batch"][case_i]
    shape, dt = tuple(case["sample_shape"]), DType(case["dtype"])
    N, B = case["samples_per_epoch"], case["batch_size"]
    sb = int(np.prod(shape)) * (4 if dt == DType.I32 else 1)
    ld = CollateLoader(DatasetSpec(SyntheticSource(0, shape, dt), N, B, shuffle_seed=0))

    def record(e, inp, tgt, crc, s):
        return e, _device_crc(inp, crc, s), tgt.cpu().numpy().copy()

    eps = (f"unix:{tmp_path}/c5b.sock", f"unix:{tmp_path}/c5a.sock")
    producer, outs = _run_facade(eps, ld, [{}] * 8, epochs, record)
    L = N // B
    frozen = {(c["epoch"], c["batch_index"]): c["crc32"]
              for c in golden["prepare_batch"] if c["name"] == case["name"]}
    assert frozen
    for got in outs:
        assert len(got) == epochs * L
    for k in range(epochs * L):
        e, bi = divmod(k, L)
        rows = {(o[k][0], o[k][1]) for o in outs}
        assert len(rows) == 1, f"consumers disagree on batch {k}"
        (ee, crc), = rows
        idx = oracle.epoch_order(N, 0, e)[bi * B:(bi + 1) * B]
        for o in outs:
            np.testing.assert_array_equal(o[k][2], idx)
        assert ee == e
        want = oracle.crc32(oracle.prepare_synthetic(0, e, idx, sb))
        assert crc == want, (e, bi)
        if (e, bi) in frozen:
            assert crc == frozen[(e, bi)], (e, bi)
    producer.close()
