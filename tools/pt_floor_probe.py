"""Per-batch floor of the persistent passthrough producer (C1, C5 video, C5
LLM): us per batch with 1 consumer and with the config's
map-and-ack consumers, at the ring depth given.  Knobs are env (read once per
process), so run one process per setting:

    TSB_PT_PER_SM=4 python tools/pt_floor_probe.py [slots] [steps]"""
import json
import os
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
from bench_configs import device_run  # noqa: E402


def main():
    import torch

    torch.cuda.set_device(0)
    from paper_2409_18749_b200 import CollateLoader, DatasetSpec, StoreSource, SyntheticSource
    from paper_2409_18749_b200.wire import DType

    slots = int(sys.argv[1]) if len(sys.argv) > 1 else 80
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
    N = 16384
    cfgs = [
        ("c1", lambda: CollateLoader(DatasetSpec(StoreSource.synthetic(0, N, (224, 224, 3),
                                                                        location="hbm"), N, 64)),
         2, 2 * 150528 * 64),
        ("c5video", lambda: CollateLoader(DatasetSpec(StoreSource.synthetic(
            0, 4096, (16, 3, 112, 112)), 4096, 16)), 8, 2 * 602112 * 16),
        ("c5llm", lambda: CollateLoader(DatasetSpec(SyntheticSource(0, (2048,), DType.I32), N,
                                                    256)), 8, 8192 * 256),
    ]
    only = os.environ.get("PROBE_ONLY", "c1,c5video,c5llm").split(",")
    for name, mk, nc, alg in cfgs:
        if name not in only:
            continue
        ld = mk()
        for consumers in ((1, nc) if os.environ.get("PROBE_BOTH") else (nc,)):
            r = device_run(ld, consumers, steps, 16, slots=slots, persistent=True)
            us = r["us_per_batch"]
            print(json.dumps({"config": name, "consumers": consumers, "slots": slots,
                              "per_sm": os.environ.get("TSB_PT_PER_SM", "default"),
                              "fence": os.environ.get("TSB_PT_FENCE", "0"), "defer": os.environ.get("TSB_PT_DEFER", "1"),
                              "us_per_batch": us, "alg_GBps": round(alg / us / 1e3, 1)}),
                  flush=True)
        del ld


if __name__ == "__main__":
    main()
