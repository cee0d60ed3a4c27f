"""Dataset model and epoch order on the host (no GPU): the reference's
TestEpochOrder / TestDatasetSpec (pkg/tests/test_pipeline.py:36-76) restated
against this package's DatasetSpec and the native epoch order
(tsb_epoch_order, the same permutation the device kernels consume)."""

import numpy as np
import pytest

from paper_2409_18749_b200 import DatasetSpec, SyntheticSource
from paper_2409_18749_b200 import dataplane as dp
from paper_2409_18749_b200.wire import DType


def synth(**kw):
    d = dict(source=SyntheticSource(seed=1, sample_shape=(64,)), samples_per_epoch=64,
             batch_size=8, shuffle_seed=3)
    d.update(kw)
    return DatasetSpec(**d)


def test_epoch_order_deterministic_and_bijective():
    a = dp.epoch_order(512, 3, 4)
    np.testing.assert_array_equal(a, dp.epoch_order(512, 3, 4))
    assert sorted(a.tolist()) == list(range(512))


def test_hundred_epochs_all_distinct():
    perms = {tuple(dp.epoch_order(1000, 3, e).tolist()) for e in range(100)}
    assert len(perms) == 100


def test_no_reshuffle_flag_and_reshuffle_differs():
    np.testing.assert_array_equal(dp.epoch_order(64, 3, 0, False), dp.epoch_order(64, 3, 5, False))
    assert dp.epoch_order(256, 3, 0).tolist() != dp.epoch_order(256, 3, 1).tolist()


def test_epoch_order_matches_oracle(oracle):
    for n, seed, epoch in ((1, 0, 0), (67, 3, 2), (16384, 0, 7)):
        np.testing.assert_array_equal(dp.epoch_order(n, seed, epoch),
                                      oracle.epoch_order(n, seed, epoch))


def test_epoch_len_drop_last():
    assert synth(samples_per_epoch=67, batch_size=8).epoch_len == 8
    assert synth(samples_per_epoch=16384, batch_size=512).epoch_len == 32


def test_batch_larger_than_epoch_is_rejected():
    with pytest.raises(ValueError):
        synth(samples_per_epoch=4, batch_size=8)
    with pytest.raises(ValueError):
        synth(batch_size=0)


def test_synthetic_sample_alignment():
    with pytest.raises(ValueError, match="multiple of 8"):
        DatasetSpec(source=SyntheticSource(sample_shape=(3,)), samples_per_epoch=8, batch_size=2)
    # (2048,) int32 tokens (C5 LLM) are 8 KB: fine
    assert synth(source=SyntheticSource(0, (2048,), DType.I32)).epoch_len == 8


@pytest.mark.gpu
def test_batch_index_bound():
    """prepare_batch(spec, prep, 0, epoch_len) raises (pipeline.py bound check;
    pkg/tests/test_pipeline.py:102-104); so does the device producer."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():  # pragma: no cover
        pytest.skip("needs a CUDA device")
    from paper_2409_18749_b200 import CollateLoader

    ld = CollateLoader(synth())
    assert len(ld) == 8
    with pytest.raises(ValueError, match="batch_index"):
        ld.produce_into(0, 0, 8)
