"""Delivered samples/s through the public API with an HBM-resident store:
TensorProducer(CollateLoader) -> K SharedLoader consumer processes (host sync,
map-and-ack).  Shows the facade's per-batch host cost next to bench.py's
native-loop value.

TSB_FR_WORK_US=W: consumer-bound mode (the reference's consumer-bound-4way,
SPEC.md:531): each consumer runs a W-us GPU step per batch (a device busy
loop, then a 4-byte read-back, as a training step's loss.item()).  Each
consumer first times the same step alone; no consumer of any API can exceed
that solo rate, so facade rate / solo rate bounds facade / native from below."""
import json
import multiprocessing as mp
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def consumer(bcast, agg, cid, n, q, sync):
    import torch

    torch.cuda.set_device(0)
    from paper_2409_18749_b200 import SharedLoader

    work_us = float(os.environ.get("TSB_FR_WORK_US", "0"))
    solo = None
    if work_us > 0:
        cycles = int(work_us * 1965)  # SM cycles at the 1965 MHz clock the bench runs at
        x = torch.zeros(1, device="cuda")

        def step(t):
            torch.cuda._sleep(cycles)
            return float(t.view(-1)[0].item())

        for _ in range(20):
            step(x)
        t0 = time.monotonic()
        for _ in range(200):
            step(x)
        solo = 200 / (time.monotonic() - t0)
    ld = SharedLoader(bcast, agg, consumer_id=cid, sync=sync)
    prof = None
    if os.environ.get("TSB_PROFILE_CONSUMER") and cid == 100:
        import cProfile

        prof = cProfile.Profile()
        prof.enable()
    ts = []
    while len(ts) < n:
        for inp, tgt in ld:
            if work_us > 0:
                step(inp)
            ts.append(time.monotonic())
            if len(ts) >= n:
                break
        if ld.finished:
            break
    ld.close()
    if prof is not None:
        import pstats

        prof.disable()
        with open(os.environ["TSB_PROFILE_CONSUMER"], "w") as fh:
            pstats.Stats(prof, stream=fh).sort_stats("tottime").print_stats(25)
    w = ts[len(ts) // 4:]
    q.put(((len(w) - 1) / (w[-1] - w[0]) if len(w) > 1 else 0.0, solo))


def main():
    import torch

    torch.cuda.set_device(0)
    from paper_2409_18749_b200 import (AugmentSpec, CollateLoader, DatasetSpec, StoreSource,
                                       TensorProducer)

    B, n = 256, int(sys.argv[1]) if len(sys.argv) > 1 else 2000
    K = int(os.environ.get("TSB_CONSUMERS", 4))
    sync = sys.argv[2] if len(sys.argv) > 2 else "host"
    store = StoreSource.synthetic(0, 16384, (224, 224, 3), location="hbm")
    ld = CollateLoader(DatasetSpec(store, 16384, B), AugmentSpec(out_dtype="float32"))
    tmp = f"/tmp/tsb-fr-{os.getpid()}"
    os.makedirs(tmp, exist_ok=True)
    b, a = f"unix:{tmp}/b.sock", f"unix:{tmp}/a.sock"
    # TSB_FR_DEVICES="0,0" + TSB_FR_FANOUT=inputs|sharded|star: the multi-ring
    # producer (one GPU here: every ring on device 0, consumers spread over them)
    devs = os.environ.get("TSB_FR_DEVICES")
    kw = {}
    if devs:
        kw = dict(devices=[int(d) for d in devs.split(",")],
                  fanout=os.environ.get("TSB_FR_FANOUT", "inputs"))
    kw["checksum"] = os.environ.get("TSB_FR_CHECKSUM", "0") == "1"
    kw["buffer_depth"] = int(os.environ.get("TSB_FR_DEPTH", 6))
    prod = TensorProducer(ld, b, a, min_consumers=K, ring_slots=8, heartbeat_timeout_s=60, **kw)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=consumer, args=(b, a, 100 + k, n, q, sync)) for k in range(K)]
    for p in ps:
        p.start()
    done, t0 = 0, None
    prof = None
    while done < n:
        for _ in prod:
            done += 1
            if done == n // 4:
                t0 = time.monotonic()
                if os.environ.get("TSB_PROFILE_PRODUCER"):
                    import cProfile

                    prof = cProfile.Profile()
                    prof.enable()
            if done >= n:
                break
    t1 = time.monotonic()
    if prof is not None:
        import pstats

        prof.disable()
        with open(os.environ["TSB_PROFILE_PRODUCER"], "w") as fh:
            pstats.Stats(prof, stream=fh).sort_stats("tottime").print_stats(30)
    prod.join(60)
    got = [q.get(timeout=300) for _ in ps]
    rates = [r for r, _ in got]
    solos = [s for _, s in got if s]
    prod.close()
    print(json.dumps({"consumer_batches_per_s": [round(r, 1) for r in rates],
                      "delivered_samples_per_s": round(sum(rates) * B, 1),
                      "producer_loop_batches_per_s": round((n - n // 4) / (t1 - t0), 1),
                      "sync": sync, "consumers": K, "checksum": kw["checksum"],
                      "buffer_depth": kw["buffer_depth"],
                      **({"work_us": float(os.environ["TSB_FR_WORK_US"]),
                          "solo_step_per_s": [round(x, 1) for x in solos],
                          "facade_over_solo": round(min(r / s for r, s in zip(rates, solos)), 4)}
                         if solos else {}),
                      **({"devices": devs, "fanout": kw["fanout"]} if devs else {})}))


if __name__ == "__main__":
    main()
