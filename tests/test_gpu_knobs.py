"""The collate kernel's tuning / A/B knobs keep it bit-exact.

The knobs (TSB_CA_R rows per item, TSB_CA_STAGES pipeline depth,
TSB_CA_ORDER item order, TSB_CA_OCC grid cap, TSB_CA_GRID absolute grid,
TSB_CA_RESIDENT resident CTAs per SM, TSB_CA_NOTMA cooperative staging,
TSB_CA_IMPL=direct staging-free kernel, TSB_CA_ST / TSB_CA_LDHINT cache
hints, TSB_BF16_FMA=0 two-rounding bf16) are read once per process, so each
configuration runs in a child process that prints the CRC-32 of the
collated batch; the parent checks it against the oracle's bytes."""

import json
import os
import subprocess
import sys
import zlib

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
H, W, C, PAD, B, N = 40, 48, 3, 6, 21, 64   # h not a multiple of any R > 8

CHILD = r"""
import json, sys, zlib
import numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2409_18749_b200 import dataplane as dp
h, w, c, pad, b, n = %d, %d, %d, %d, %d, %d
sb = h * w * c
store = torch.empty(n * sb, dtype=torch.uint8, device="cuda")
dp.make_store(store, 5, n, sb)
idx = torch.from_numpy(dp.epoch_order(n, 0, 2)[:b].copy()).cuda()
scale, bias = dp.norm_consts()
res = {}
for kind, ob in ((0, 1), (1, 4), (2, 2)):
    out = torch.empty(b * c * h * w * ob, dtype=torch.uint8, device="cuda")
    dp.collate_augment(store, idx, b, h, w, c, pad, True, 9, 2, kind, out, scale=scale, bias=bias)
    res[kind] = zlib.crc32(out.cpu().numpy().tobytes())
print(json.dumps(res))
""" % (H, W, C, PAD, B, N)

KNOBS = [
    {},
    {"TSB_CA_R": "1", "TSB_CA_STAGES": "1"},
    {"TSB_CA_R": "2", "TSB_CA_STAGES": "4", "TSB_CA_ORDER": "blocked"},
    {"TSB_CA_R": "32", "TSB_CA_STAGES": "2", "TSB_CA_OCC": "1"},
    {"TSB_CA_RESIDENT": "3", "TSB_CA_ORDER": "blocked"},
    {"TSB_CA_R": "7", "TSB_CA_STAGES": "3", "TSB_CA_GRID": "5"},
    {"TSB_CA_NOTMA": "1"},
    {"TSB_CA_IMPL": "direct"},
    {"TSB_CA_ST": "plain", "TSB_CA_LDHINT": "0"},
    {"TSB_BF16_FMA": "0"},
]


@pytest.fixture(scope="module")
def want(oracle):
    store = oracle.make_store(5, N, H * W * C)
    idx = oracle.epoch_order(N, 0, 2)[:B]
    scale, bias = oracle.norm_consts()
    return {kind: zlib.crc32(oracle.collate_augment(store, idx, H, W, C, PAD, True, 9, 2, kind,
                                                    scale, bias, nthreads=4).tobytes())
            for kind in (0, 1, 2)}


@pytest.mark.parametrize("knobs", KNOBS, ids=lambda k: ",".join(f"{a[7:]}={v}" for a, v in
                                                               k.items()) or "defaults")
def test_collate_knobs_bit_exact(want, knobs):
    env = dict(os.environ, **knobs)
    r = subprocess.run([sys.executable, "-c", CHILD, ROOT], env=env, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    got = {int(k): v for k, v in json.loads(r.stdout.strip().splitlines()[-1]).items()}
    assert got == want
