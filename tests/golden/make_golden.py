"""Generate tests/golden/golden.json by RUNNING THE REFERENCE in this container.

    PYTHONPATH is set up below from /root/reference (read-only); numba caches
    go to /tmp.  Run:  python tests/golden/make_golden.py

The reference cannot travel to the GPU box, so its outputs are frozen here
as small fixtures; tests pin the CPU oracle (oracle/) and the CUDA path to
them.  Every entry names the reference function that produced it.
"""

from __future__ import annotations

import json
import os
import sys
import tempfile
import zlib

REF = "/root/reference/pkg"
sys.path[:0] = [f"{REF}/src", f"{REF}/frontend/src"]
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")

import numpy as np  # noqa: E402

from batchsocket import kernels, payload, pipeline, wire  # noqa: E402
from batchsocket.pipeline import DatasetSpec, DirectorySource, PrepSpec, SyntheticSource  # noqa: E402
from sharedloader import abi as facade_abi  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")


def crc(b) -> int:
    return zlib.crc32(bytes(b)) & 0xFFFFFFFF


def main() -> None:
    g: dict = {"generator": "tests/golden/make_golden.py", "reference": REF,
               "kernels_backend": kernels.BACKEND}

    # kernels.py:40-45
    xs = [0, 1, 2, 0x9E3779B97F4A7C15, (1 << 64) - 1, 0x0123456789ABCDEF, 42]
    g["mix64"] = [[x, kernels.mix64(x)] for x in xs]
    # kernels.py:48-53
    g["derive_key"] = [[s, e, i, kernels.derive_key(s, e, i)]
                       for s in (0, 1, 12345) for e in (0, 1, 7)
                       for i in (0, 1, 0x53485546, 1000003)]
    # kernels.py:170-178
    perms = []
    for n, key in [(0, 5), (1, 5), (2, 5), (10, 42), (17, 3), (16, kernels.derive_key(0, 0, 0x53485546)),
                   (1000, 0xDEADBEEF), (100000, 7)]:
        p = kernels.permutation(n, key)
        entry = {"n": n, "key": key, "crc_i64": crc(p.astype("<i8").tobytes()),
                 "head": p[:32].tolist()}
        if n <= 1000:
            entry["perm"] = p.tolist()
        perms.append(entry)
    g["permutation"] = perms
    # kernels.py:158-167
    keys = np.array([kernels.derive_key(0, 0, 0), kernels.derive_key(0, 0, 1), 7], dtype=np.uint64)
    out = np.empty(3 * 5, dtype=np.uint64)
    kernels.fill_batch(out, keys, 5)
    g["fill_batch"] = {"keys": [int(k) for k in keys], "wps": 5, "words": [int(w) for w in out]}

    # pipeline.py:113-123 epoch_order
    orders = []
    for n, seed, epoch, resh in [(1024, 0, 0, True), (1024, 0, 1, True), (2048, 0, 0, True),
                                 (16384, 0, 0, True), (16384, 0, 1, True), (16384, 0, 5, False),
                                 (64, 3, 2, True)]:
        spec = DatasetSpec(SyntheticSource(seed=0, sample_shape=(8,)), n, 1, shuffle_seed=seed,
                           reshuffle_each_epoch=resh)
        o = pipeline.epoch_order(spec, epoch)
        orders.append({"n": n, "shuffle_seed": seed, "epoch": epoch, "reshuffle": resh,
                       "crc_i64": crc(o.astype("<i8").tobytes()), "head": o[:16].tolist()})
    g["epoch_order"] = orders

    # pipeline.py:158-213 prepare_batch, synthetic source
    batches = []
    cases = [
        ("img_b64", (224, 224, 3), wire.DType.U8, 64, 1024, 0, [(0, 0), (0, 3), (1, 0), (1, 15)]),
        ("img_b256", (224, 224, 3), wire.DType.U8, 256, 2048, 0, [(0, 0), (2, 7)]),
        ("llm", (2048,), wire.DType.I32, 256, 1024, 0, [(0, 0), (1, 3)]),
        ("video", (16, 3, 112, 112), wire.DType.U8, 16, 256, 0, [(0, 0), (3, 15)]),
        ("small_seed9", (64,), wire.DType.U8, 8, 67, 9, [(0, 0), (4, 7)]),
    ]
    for name, shape, dt, bsz, n, seed, eb in cases:
        spec = DatasetSpec(SyntheticSource(seed=seed, sample_shape=shape, dtype=dt), n, bsz,
                           shuffle_seed=seed)
        for epoch, bi in eb:
            dtype, bshape, buf = pipeline.prepare_batch(spec, PrepSpec(), epoch, bi)
            order = pipeline.epoch_order(spec, epoch)
            batches.append({
                "name": name, "sample_shape": list(shape), "dtype": int(dtype), "batch_size": bsz,
                "samples_per_epoch": n, "seed": seed, "shuffle_seed": seed, "epoch": epoch,
                "batch_index": bi, "epoch_len": spec.epoch_len, "shape": list(bshape),
                "indices": order[bi * bsz:(bi + 1) * bsz].tolist(), "crc32": crc(buf),
                "nbytes": len(buf), "head8": list(bytes(buf[:8])), "sum": int(np.frombuffer(buf, np.uint8).sum(dtype=np.uint64)),
            })
    g["prepare_batch"] = batches

    # pipeline.py:139-155,190-210 directory source
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "ds")
        pipeline.write_directory_dataset(path, num_samples=64, sample_bytes=4096, seed=5)
        spec = DatasetSpec(DirectorySource(path, 4096), 64, 16, shuffle_seed=11)
        dirb = []
        for epoch, bi in [(0, 0), (0, 3), (1, 0), (2, 2)]:
            _, _, buf = pipeline.prepare_batch(spec, PrepSpec(), epoch, bi)
            order = pipeline.epoch_order(spec, epoch)
            dirb.append({"epoch": epoch, "batch_index": bi,
                         "indices": order[bi * 16:(bi + 1) * 16].tolist(), "crc32": crc(buf)})
        files = [crc(open(os.path.join(path, f"sample-{i:08d}.bin"), "rb").read()) for i in range(64)]
    g["directory"] = {"num_samples": 64, "sample_bytes": 4096, "seed": 5, "batch_size": 16,
                      "shuffle_seed": 11, "file_crc32": files, "batches": dirb}

    # rebatch invariance: epoch order is independent of batch size
    reb = []
    n = 2048
    for bsz in (64, 128, 256, 512):
        spec = DatasetSpec(SyntheticSource(seed=0, sample_shape=(8,)), n, bsz)
        crcs = []
        for bi in range(min(4, spec.epoch_len)):
            _, _, buf = pipeline.prepare_batch(spec, PrepSpec(), 1, bi)
            crcs.append(crc(buf))
        reb.append({"batch_size": bsz, "epoch_len": spec.epoch_len, "epoch": 1, "crc32": crcs})
    spec64 = DatasetSpec(SyntheticSource(seed=0, sample_shape=(8,)), n, 64)
    spec512 = DatasetSpec(SyntheticSource(seed=0, sample_shape=(8,)), n, 512)
    cat = b"".join(bytes(pipeline.prepare_batch(spec64, PrepSpec(), 1, j)[2]) for j in range(8))
    big = bytes(pipeline.prepare_batch(spec512, PrepSpec(), 1, 0)[2])
    g["rebatch"] = {"samples_per_epoch": n, "sample_shape": [8], "cases": reb,
                    "concat64_eq_512": cat == big}

    # wire.py:199-246 frozen frames
    frames = {
        "join": wire.Join(123456789, 1),
        "welcome": wire.Welcome(7, 3, 1000, 12, 2, 1),
        "announce_imagenet": wire.Announce(2, 9, "tsk-1234-2-9", 512 * 3 * 224 * 224 * 4,
                                           wire.DType.F32, (512, 3, 224, 224), 0xABCD1234),
        "announce_scalar": wire.Announce(0, 0, "x", 8, wire.DType.I64, (), 0),
        "ack": wire.Ack(7, 0, 42),
        "heartbeat": wire.Heartbeat(5, 123456),
        "epoch_start": wire.EpochStart(4, 250),
        "epoch_end": wire.EpochEnd(4),
        "bye": wire.Bye(99),
        "shutdown": wire.Shutdown(),
    }
    g["frames"] = {k: wire.encode_message(m).hex() for k, m in frames.items()}

    # payload.py:165-248 segment header (80 bytes)
    data = np.arange(2 * 3 * 4, dtype=np.float32).reshape(2, 3, 4)
    p, desc = payload.create_segment(3, 17, wire.DType.F32, (2, 3, 4), data.tobytes(),
                                     reserved=b"abc", name=f"golden-{os.getpid()}")
    try:
        v = payload.map_segment(desc.segment_name)
        raw = bytes(v._shm.buf[:payload.HEADER_SIZE])
        v.close()
    finally:
        payload.release_segment(p)
    g["segment_header"] = {"epoch": 3, "batch_index": 17, "dtype": 3, "shape": [2, 3, 4],
                           "reserved": "abc", "payload_crc32": crc(data.tobytes()), "hex": raw.hex()}
    # sl/abi.py:303-306 pair encoding
    g["pair_reserved"] = facade_abi.pack_pair_reserved(3, 4, 2, 1, 256 * 3 * 224 * 224 * 4).hex()
    g["facade_frames"] = {
        "announce": facade_abi.encode(facade_abi.Announce_(0, 5, "tsk-1-0-5", 100, 0, (100,), 77)).hex(),
        "ack": facade_abi.encode(facade_abi.Ack_(7, 0, 42)).hex(),
    }
    # wire.py:170-172 known answers
    g["crc32"] = [[b.hex(), crc(b)] for b in (b"", b"123456789", b"a", bytes(range(256)), b"\xff" * 1000)]

    with open(OUT, "w") as fh:
        json.dump(g, fh, indent=1, sort_keys=True)
    print(f"wrote {OUT} ({os.path.getsize(OUT)} bytes)")


if __name__ == "__main__":
    main()
