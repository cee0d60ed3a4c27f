"""Where does per-batch pipeline time go?  Producer rate for the C2 batch with
0 consumers, in-process consumer streams, and consumer processes."""
import json
import multiprocessing as mp
import sys

import torch

sys.path.insert(0, ".")
from bench import device_consumer  # noqa: E402
from paper_2409_18749_b200 import AugmentSpec, CollateLoader, DatasetSpec, StoreSource  # noqa: E402
from paper_2409_18749_b200 import dataplane as dp  # noqa: E402
from paper_2409_18749_b200.ring import DeviceRing, consume_range, produce_range  # noqa: E402

import os
B, N, K, Wm = 256, 16384, 48, 8
S = int(os.environ.get("SLOTS", 8))
STRIDE = int(os.environ.get("STRIDE", 1))
ld = None


def host_consumer(handle, ctl, slots, slot_bytes, mc, cursor, n, q):
    import torch
    torch.cuda.set_device(0)
    from paper_2409_18749_b200.ring import DeviceRing
    ring = DeviceRing.import_handle(handle, slots, slot_bytes, mc, ctl)
    q.put("ready")
    for seq in range(1, n + 1):
        ring.host_wait_ready((seq - 1) % slots, seq)
        ring.host_ack(cursor, seq)
    q.put("done")


def run(mode, ncons, control="device"):
    ring = DeviceRing(S, ld.batch_nbytes, max(1, ncons), control=control)
    s = torch.cuda.Stream()
    procs, threads = [], []
    q = None
    if mode == "proc":
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        procs = [ctx.Process(target=device_consumer, args=(0, ring.export(), S, ld.batch_nbytes, ncons, k, Wm, K, q, ring.control_name))
                 for k in range(ncons)]
        for p in procs:
            p.start()
        for _ in procs:
            q.get(timeout=120)
    elif mode == "hproc":
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        procs = [ctx.Process(target=host_consumer, args=(ring.export(), ring.control_name, S, ld.batch_nbytes, ncons, k, Wm + K, q))
                 for k in range(ncons)]
        for p in procs:
            p.start()
        for _ in procs:
            q.get(timeout=120)
    elif mode == "thread":
        streams = [torch.cuda.Stream() for _ in range(ncons)]
        for k in range(ncons):
            consume_range(ring, k, 1, Wm + K, stream=streams[k])
    live = list(range(ncons)) if mode != "none" else []
    a = ld.produce_args(0)
    a.wait_stride = STRIDE
    a.gate = int(os.environ.get("GATE", 0)) if control == "host" else 0
    produce_range(ring, a, 1, 0, Wm, live, stream=s)
    s.synchronize()
    e0, e1 = dp.DeviceEvent(), dp.DeviceEvent()
    e0.record(s)
    produce_range(ring, a, Wm + 1, Wm, K, live, stream=s)
    e1.record(s)
    s.synchronize()
    ms = e0.elapsed_ms(e1)
    for _ in procs:
        q.get(timeout=120)
    for p in procs:
        p.join()
    torch.cuda.synchronize()
    ring.close()
    return round(B * K / (ms / 1e3)), round(ms / K * 1000, 1)


if __name__ == "__main__":
    torch.cuda.set_device(0)
    store = StoreSource.synthetic(0, N, (224, 224, 3))
    ld = CollateLoader(DatasetSpec(store, N, B),
                       AugmentSpec(out_dtype=sys.argv[2] if len(sys.argv) > 2 else "float32"))
    res = {}
    for mode, n, ctl in [("none", 0, "host"), ("hproc", 4, "host")]:
        res[f"{mode}{n}-{ctl}"] = run(mode, n, ctl)
        print(mode, n, ctl, res[f"{mode}{n}-{ctl}"], flush=True)
    print(json.dumps(res))
