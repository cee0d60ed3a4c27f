"""The UNMODIFIED reference CPU data plane, timed on this host's cores.

BASELINE.md §4: beside every GPU measurement, run the reference's own
`batchsocket.harness.run_scenario` (bs/harness.py:411) in shared mode from
`baseline/_ref` -- a git-ignored `pip install --target` of /root/reference
that travels to the GPU box with the snapshot -- at each config's sample
shape, batch size and consumer count, with compute_us = pace_us = 0,
prep_cost_us_per_sample = 0, workers = nproc, and report the reference's own
formula: per-consumer (n-1)/(t_last-t_first)*batch averaged over epochs
(bs/harness.py:611-617), summed over consumers (:574).

    python tools/ref_cpu_bench.py [--only c1,c2,c5video,c5llm] [--epoch-len 60]

This is a measurement tool, not part of the product: nothing in the package
imports it, and bench.py's reference arm stays the oracle port.
The reference delivers the collated u8 batch (no crop/flip/normalise exists
in it), so its C2 line is the u8 shape.
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

CONFIGS = {  # name: (sample_bytes, batch_size, consumers)
    "c1": (224 * 224 * 3, 64, 2),
    "c2": (224 * 224 * 3, 256, 4),
    "c5video": (16 * 3 * 112 * 112, 16, 8),
    "c5llm": (2048 * 4, 256, 8),
}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="c1,c2,c5video,c5llm")
    ap.add_argument("--epoch-len", type=int, default=60)
    ap.add_argument("--epochs", type=int, default=2)
    args = ap.parse_args()
    if not os.path.isdir(os.path.join(REF, "batchsocket")):
        print(json.dumps({"unavailable": "baseline/_ref has no reference install"}))
        return
    # the scenario's child processes run `python -m batchsocket`, so the
    # install must be importable through the environment, not just sys.path
    os.environ["PYTHONPATH"] = REF + os.pathsep + os.environ.get("PYTHONPATH", "")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/tsb-ref-numba")
    sys.path.insert(0, REF)
    from batchsocket.harness import ConsumerLoad, ScenarioSpec, run_scenario

    nproc = os.cpu_count() or 1
    for name in args.only.split(","):
        sb, b, k = CONFIGS[name]
        spec = ScenarioSpec(name=f"ref-{name}", consumers=[ConsumerLoad() for _ in range(k)],
                            mode="shared", workers=nproc, epochs=args.epochs,
                            epoch_len=args.epoch_len, batch_size=b, sample_bytes=sb,
                            prep_cost_us_per_sample=0, oracle_check=False, timeout_s=900)
        rep = run_scenario(spec)
        print(json.dumps({
            "config": name, "impl": "reference (baseline/_ref, unmodified, run_scenario shared)",
            "sample_bytes": sb, "batch_size": b, "consumers": k, "workers": nproc,
            "epochs": args.epochs, "epoch_len": args.epoch_len,
            "aggregate_samples_s": round(rep.aggregate_samples_s, 1),
            "per_consumer_samples_s": [round(r, 1) for r in rep.per_consumer_samples_s],
            "wall_s": round(rep.wall_seconds, 2), "nproc": nproc, "cpu": cpu_model()}),
            flush=True)


if __name__ == "__main__":
    main()
