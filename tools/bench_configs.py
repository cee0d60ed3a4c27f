"""Per-config measurements on ONE B200 (BASELINE.json configs C1, C2-bf16, C4,
C5), next to the reference CPU numbers of SURVEY.md §6 / BASELINE.md §2.

    python tools/bench_configs.py [--steps K] [--only c1,c4,...]

Device-resident runs use the native producer loop (host flow gate, fused
publish, PDL chain) with map-and-ack consumer processes (bs/cli.py:252-258);
C4 runs heterogeneous SharedLoader consumers through the facade (rebatch).
Prints one JSON line per config.  C3 and the multi-GPU halves of C4/C5 need
several GPUs: see bench.py --gpus N and tools/nccl_broadcast_compare.py.
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import host_consumer  # noqa: E402

# the UNMODIFIED reference (baseline/_ref, run_scenario shared mode) on the GPU
# box's 16 host cores, aggregate delivered samples/s (profiles/r1/ref_cpu_gpu_host.jsonl)
REF = {"c1": 19050.7, "c2_shape_u8": 35139.1, "c5_llm_k8": 938897.3, "c5_video_k8": 18014.0}
REF_SOURCE = "profiles/r1/ref_cpu_gpu_host.jsonl (unmodified reference, 16 host cores)"
L2_BYTES = 126 * 2**20
# persistent passthrough: epochs per launch (TSB_EPOCHS_PER_LAUNCH; 1 = a launch per epoch)
EPOCHS_PER_LAUNCH = int(os.environ.get("TSB_EPOCHS_PER_LAUNCH", "1"))


def hbm_line(r: dict, sample_bytes: int, slots: int, slot_bytes: int, rw: int = 2) -> dict:
    """Passthrough roofline: each produced sample is read once and written
    once (rw = 2 x sample_bytes; rw = 1 for the synthetic source, generated
    in the kernel); the ring must exceed L2 for the writes to reach HBM."""
    import json as _j
    import os as _o

    peak = 6532.2
    try:
        with open(_o.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peak = float(_j.load(fh)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        pass
    produced = r["value"] / r["consumers"]
    gbs = produced * rw * sample_bytes / 1e9
    return {"hbm_alg_gbs": round(gbs, 1), "alg_bytes_per_sample": rw * sample_bytes, "hbm_frac": round(gbs / peak, 4), "hbm_peak_gbs": peak,
            "ring_bytes": slots * slot_bytes, "ring_exceeds_l2": slots * slot_bytes > L2_BYTES}


def device_run(loader, n_consumers, steps, warmup, slots=8, persistent=False):
    """value: delivered samples/s of the native producer loop (device time)."""
    import torch

    from paper_2409_18749_b200 import dataplane as dp
    from paper_2409_18749_b200._lib import GATE_HOST
    from paper_2409_18749_b200.ring import DeviceRing, produce_range

    ring = DeviceRing(slots, loader.batch_nbytes, n_consumers, control="host")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=host_consumer, args=(0, ring.export(), ring.control_name, slots,
                                                      loader.batch_nbytes, n_consumers, k, warmup,
                                                      steps, q))
             for k in range(n_consumers)]
    for p in procs:
        p.start()
    for _ in procs:
        q.get(timeout=300)
    L = len(loader)
    s = torch.cuda.Stream()

    # persistent passthrough: one launch may span several epochs (short epochs,
    # e.g. C5 LLM's 64 batches, would otherwise pay a launch + host round each)
    multi = persistent and loader.augment is None and EPOCHS_PER_LAUNCH > 1

    def produce(seq0, n):
        done = 0
        while done < n:
            q0 = seq0 + done
            ep, bi = divmod(q0 - 1, L)
            if multi:
                k = min(EPOCHS_PER_LAUNCH, -(-(bi + n - done) // L))
                m = min(n - done, k * L - bi)
                a = loader.produce_args_epochs(ep, k)
            else:
                m = min(n - done, L - bi)
                a = loader.produce_args(ep)
            a.gate = GATE_HOST
            a.persistent = int(persistent)
            produce_range(ring, a, q0, bi, m, list(range(n_consumers)), stream=s)
            done += m

    produce(1, warmup)
    s.synchronize()
    e0, e1 = dp.DeviceEvent(), dp.DeviceEvent()
    e0.record(s)
    produce(warmup + 1, steps)
    e1.record(s)
    s.synchronize()
    ms = e0.elapsed_ms(e1)
    for _ in procs:
        q.get(timeout=300)
    for p in procs:
        p.join(60)
    ring.close()
    b = loader.dataset.batch_size
    return {"produced_batches_per_s": round(steps / (ms / 1e3), 1),
            "value": round(n_consumers * b * steps / (ms / 1e3), 1),
            "us_per_batch": round(1e3 * ms / steps, 2), "consumers": n_consumers}


def c4_consumer(bcast, agg, cid, b, epochs, q):
    import torch

    torch.cuda.set_device(0)
    from paper_2409_18749_b200 import SharedLoader

    loader = SharedLoader(bcast, agg, consumer_id=cid, batch_size=b, sync="host")
    q.put(("ready", cid))
    rates, n = [], 0
    for _ in range(epochs):
        times = []
        for inp, tgt in loader:
            times.append(time.monotonic())
            n += 1
        if len(times) > 1:  # the reference's per-epoch rate (bs/cli.py:220-236)
            rates.append((len(times) - 1) / (times[-1] - times[0]) * b)
    loader.close()
    rate = sum(rates) / len(rates) if rates else 0.0  # mean over epochs, bs/harness.py:611-617
    q.put(("done", cid, b, rate, n))


def c4(epochs=5):
    """Heterogeneous consumers b in {64,128,256,512} (2 each) on one producer
    of B=512 bf16 batches: every consumer gets the reference's batches for its
    own b (zero-copy windows); per-consumer rate by the reference formula."""
    from paper_2409_18749_b200 import (AugmentSpec, CollateLoader, DatasetSpec, StoreSource,
                                       TensorProducer)

    N = 16384
    store = StoreSource.synthetic(0, N, (224, 224, 3), location="hbm")
    ld = CollateLoader(DatasetSpec(store, N, 512), AugmentSpec(out_dtype="bfloat16"))
    tmp = f"/tmp/tsb-c4-{os.getpid()}"
    os.makedirs(tmp, exist_ok=True)
    bcast, agg = f"unix:{tmp}/b.sock", f"unix:{tmp}/a.sock"
    sizes = [64, 64, 128, 128, 256, 256, 512, 512]
    producer = TensorProducer(ld, bcast, agg, min_consumers=len(sizes), ring_slots=6,
                              heartbeat_timeout_s=60)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=c4_consumer, args=(bcast, agg, 500 + i, b, epochs, q))
             for i, b in enumerate(sizes)]
    for p in procs:
        p.start()
    t0 = time.monotonic()
    for _ in range(epochs):
        for _ in producer:
            pass
    producer.join(60)
    wall = time.monotonic() - t0
    rates = []
    while len(rates) < len(sizes):
        m = q.get(timeout=300)
        if m[0] == "done":
            rates.append(m[2:])
    for p in procs:
        p.join(60)
    producer.close()
    return {"value": round(sum(r[1] for r in rates), 1),
            "per_batch_size": {str(b): round(sum(r[1] for r in rates if r[0] == b), 1)
                               for b in sorted(set(sizes))},
            "batches_per_consumer": {str(b): sorted({r[2] for r in rates if r[0] == b})
                                     for b in sorted(set(sizes))},
            "wall_s": round(wall, 2), "epochs": epochs, "producer_batch": 512}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=512)
    ap.add_argument("--warmup", type=int, default=16)
    ap.add_argument("--only", default="c1,c2bf16,c5video,c5llm,c4native,c4")
    ap.add_argument("--slots", type=int, default=8,
                    help="ring slots for the passthrough configs (C1, C5); > L2 for HBM fractions")
    ap.add_argument("--persistent", action="store_true",
                    help="passthrough configs (C1, C5) as one persistent launch per range")
    args = ap.parse_args()
    import torch

    torch.cuda.set_device(0)
    from paper_2409_18749_b200 import (AugmentSpec, CollateLoader, DatasetSpec, StoreSource,
                                       SyntheticSource)
    from paper_2409_18749_b200.wire import DType

    which = args.only.split(",")
    K, Wm = args.steps, args.warmup
    N = 16384
    if "c1" in which:
        store = StoreSource.synthetic(0, N, (224, 224, 3), location="hbm")
        ld = CollateLoader(DatasetSpec(store, N, 64))
        r = device_run(ld, 2, K, Wm, slots=args.slots, persistent=args.persistent)
        r.update(config="C1: 224x224x3 u8 passthrough (DirectorySource gather), B=64, 2 consumers"
                 + (" [persistent]" if args.persistent else ""),
                 reference_cpu=REF["c1"], reference_source=REF_SOURCE,
                 **hbm_line(r, 150528, args.slots, ld.batch_nbytes))
        print(json.dumps(r), flush=True)
        del store, ld
    if "c2bf16" in which:
        store = StoreSource.synthetic(0, N, (224, 224, 3), location="hbm")
        ld = CollateLoader(DatasetSpec(store, N, 256), AugmentSpec(out_dtype="bfloat16"))
        r = device_run(ld, 4, K, Wm)
        r.update(config="C2 shape, bf16 NCHW (crop/flip/normalise), B=256, 4 IPC consumers",
                 alg_GBps=round(r["value"] / 4 * (150528 + 301056) / 1e9, 1))
        print(json.dumps(r), flush=True)
        del store, ld
    if "c5video" in which:
        ld = CollateLoader(DatasetSpec(StoreSource.synthetic(0, 4096, (16, 3, 112, 112)), 4096,
                                       16))
        r = device_run(ld, 8, K, Wm, slots=args.slots, persistent=args.persistent)
        r.update(config="C5 video: (16,3,112,112) u8 clips, B=16, 8 consumers (one GPU)"
                 + (" [persistent]" if args.persistent else ""),
                 reference_cpu=REF["c5_video_k8"], reference_source=REF_SOURCE,
                 **hbm_line(r, 602112, args.slots, ld.batch_nbytes))
        print(json.dumps(r), flush=True)
        del ld
    if "c5llm" in which:
        ld = CollateLoader(DatasetSpec(SyntheticSource(0, (2048,), DType.I32), N, 256))
        r = device_run(ld, 8, K, Wm, slots=args.slots, persistent=args.persistent)
        r.update(config="C5 LLM: (2048,) int32 tokens (SyntheticSource on device), B=256, "
                        "8 consumers (one GPU)" + (" [persistent]" if args.persistent else ""),
                 reference_cpu=REF["c5_llm_k8"], reference_source=REF_SOURCE,
                 **hbm_line(r, 8192, args.slots, ld.batch_nbytes, rw=1))
        print(json.dumps(r), flush=True)
        del ld
    if "jpeg" in which:
        import io

        import numpy as np
        from PIL import Image

        from paper_2409_18749_b200 import JpegSource

        rng = np.random.default_rng(0)
        yy, xx = np.mgrid[0:224, 0:224].astype(np.float32)
        files = []
        for i in range(1024):
            f = rng.uniform(0.02, 0.2, 3)
            img = np.stack([127 + 100 * np.sin(f[c] * xx + i) * np.cos(f[c] * yy)
                            for c in range(3)], -1)
            img = np.clip(img + rng.normal(0, 6, img.shape), 0, 255).astype(np.uint8)
            b = io.BytesIO()
            Image.fromarray(img).save(b, format="JPEG", quality=90)
            files.append(b.getvalue())
        src = JpegSource(files, 224, 224)
        ld = CollateLoader(DatasetSpec(src, 1024, 256), AugmentSpec(out_dtype="bfloat16"))
        r = device_run(ld, 4, min(K, 64), Wm)
        r.update(config="JPEG store (1024 x 224x224 q90 4:2:0, ~%d KB/file) -> nvJPEG batched "
                        "decode (%s) -> crop/flip/normalise bf16, B=256, 4 consumers"
                        % (sum(map(len, files)) // len(files) // 1024,
                           src.decoder(0, 256).backend))
        print(json.dumps(r), flush=True)
    if "c4native" in which:
        # the data plane under C4: one B=512 bf16 producer, 8 map-and-ack consumers.
        # A consumer with b in {64,128,256,512} reads b-sample zero-copy windows of
        # the slot (ledger.rebatch_window_plan) and releases the slot after its last
        # window there, so per slot it receives the same 512 samples.
        store = StoreSource.synthetic(0, N, (224, 224, 3), location="hbm")
        ld = CollateLoader(DatasetSpec(store, N, 512), AugmentSpec(out_dtype="bfloat16"))
        r = device_run(ld, 8, K, Wm)
        r.update(config="C4 data plane (one GPU): B=512 bf16 slots, 8 map-and-ack consumers "
                        "(b=64..512 read zero-copy windows of each slot)")
        print(json.dumps(r), flush=True)
        del store, ld
    if "c4" in which:
        r = c4()
        r.update(config="C4 (one GPU): consumers with b=64/128/256/512 (2 each) on one producer "
                        "of B=512 bf16, facade rebatch, host-synced consumer processes")
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
