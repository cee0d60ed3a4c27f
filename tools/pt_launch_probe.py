"""Per-launch device time of the persistent passthrough producer against the
whole range's time: are the gaps between epoch launches or inside them?
(C1 shape: B=64 224x224x3 u8 gather, 80 slots, 2 map-and-ack consumers.)

    python tools/pt_launch_probe.py [epochs]"""
import json
import multiprocessing as mp
import sys
import time

sys.path.insert(0, ".")
sys.path.insert(0, "tools")


def main():
    import torch

    from bench import host_consumer
    from paper_2409_18749_b200 import CollateLoader, DatasetSpec, StoreSource
    from paper_2409_18749_b200 import dataplane as dp
    from paper_2409_18749_b200._lib import GATE_HOST
    from paper_2409_18749_b200.ring import DeviceRing, produce_range

    torch.cuda.set_device(0)
    E = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    N, B, S, NC = 16384, 64, 80, 2
    ld = CollateLoader(DatasetSpec(StoreSource.synthetic(0, N, (224, 224, 3), location="hbm"),
                                   N, B))
    L = len(ld)
    ring = DeviceRing(S, ld.batch_nbytes, NC, control="host")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=host_consumer, args=(0, ring.export(), ring.control_name, S,
                                                      ld.batch_nbytes, NC, k, 0, E * L, q))
             for k in range(NC)]
    for p in procs:
        p.start()
    for _ in procs:
        q.get(timeout=300)
    s = torch.cuda.Stream()
    evs, host_us = [], []
    t_all0 = dp.DeviceEvent()
    t_all0.record(s)
    for e in range(E):
        t0 = time.perf_counter()
        a = ld.produce_args(e)
        a.gate = GATE_HOST
        a.persistent = 1
        e0, e1 = dp.DeviceEvent(), dp.DeviceEvent()
        e0.record(s)
        produce_range(ring, a, e * L + 1, 0, L, list(range(NC)), stream=s)
        e1.record(s)
        host_us.append((time.perf_counter() - t0) * 1e6)
        evs.append((e0, e1))
    t_all1 = dp.DeviceEvent()
    t_all1.record(s)
    s.synchronize()
    per = [a.elapsed_ms(b) * 1e3 for a, b in evs]
    gaps = [evs[i - 1][1].elapsed_ms(evs[i][0]) * 1e3 for i in range(1, E)]
    total = t_all0.elapsed_ms(t_all1) * 1e3
    for _ in procs:
        q.get(timeout=300)
    for p in procs:
        p.join(60)
    print(json.dumps({"batches_per_launch": L, "launch_us": [round(x, 1) for x in per],
                      "gap_us": [round(x, 1) for x in gaps],
                      "host_enqueue_us": [round(x, 1) for x in host_us],
                      "us_per_batch_total": round(total / (E * L), 3),
                      "us_per_batch_in_launch": round(sum(per) / (E * L), 3)}))
    ring.close()


if __name__ == "__main__":
    main()
