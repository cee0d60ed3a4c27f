"""bench.py's reference arm runs on CPU: its JSON line carries the contract
keys (impl, metric/value/unit, cpu_baseline with kind/cores/sample, e2e with
zero host<->device bytes) and finishes quickly with a bounded sample."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "2", "--warmup", "3"], capture_output=True, text=True,
                         timeout=600, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "samples/s" and d["value"] > 0
    assert d["metric"].startswith("delivered samples/sec") and d["higher_is_better"] is True
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": "samples/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert d["config"]["workload"].startswith("C2")


def test_warmup_floor_enforced():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--warmup", "2"],
                         capture_output=True, text=True, timeout=120, cwd=ROOT)
    assert out.returncode != 0 and "warmup" in out.stderr


def _reduce_worker(rank, world, port, q):
    import torch.distributed as dist

    import bench

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        r, w, lr = bench.dist_env()
        ms = [3.5, 7.25][rank]  # per-rank device time of the timed region
        q.put((rank, (r, w, lr), bench.reduce_over_ranks(ms, "max", "gloo"),
               bench.reduce_over_ranks(1000.0 * (rank + 1), "sum", "gloo")))
    finally:
        dist.destroy_process_group()


def test_multi_rank_timing_is_max_over_ranks_gloo_world2():
    """bench.py at N > 1: every rank reads its rank from the env, the timed
    region is the max over ranks, e2e throughput is summed over ranks."""
    import multiprocessing as mp
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_reduce_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = {m[0]: m[1:] for m in (q.get(timeout=120) for _ in ps)}
    for p in ps:
        p.join(30)
    for r in (0, 1):
        assert res[r] == ((r, 2, r), 7.25, 3000.0)


def test_common_window_rate():
    """e2e aggregate over the window every consumer was fetching in: a
    consumer that started late does not inflate the others' count, and a
    consumer's own start-up skew is cut off (bench.common_window_rate)."""
    import bench

    B = bench.B
    stamps = {
        1: [0.0 + 0.01 * i for i in range(101)],   # 0.00 .. 1.00
        2: [0.5 + 0.01 * i for i in range(101)],   # 0.50 .. 1.50 (late start)
    }
    rate, window, n = bench.common_window_rate(stamps)
    assert abs(window - 0.5) < 1e-9
    # window (0.5, 1.0]: 50 fetches each
    assert n == 100
    assert abs(rate - 100 * B / 0.5) < 1e-6 * rate
    assert bench.common_window_rate({1: [0.0, 1.0], 2: [2.0, 3.0]}) == (0.0, 0.0, 0)
