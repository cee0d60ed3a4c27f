"""Benchmark of the shared-loading hot path on B200 (prints ONE JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...       (one rank per GPU)

Workload (BASELINE.json configs[1], "C2"): 1 producer + 4 consumers on one
B200 via CUDA IPC zero copy, ResNet-50-shaped batches of 256: a
DirectorySource-equivalent store of 16,384 uint8 224x224x3 samples
(SplitMix64, the reference RNG), the reference epoch shuffle, then the fused
collate/augment (RandomCrop pad 16 + HFlip with params from the reference RNG,
ImageNet normalise) to float32 NCHW written into the device ring; consumers in
other processes map the ring over CUDA IPC and release slots with
device-counted acks.  A step = one batch of 256 produced and delivered to all
4 consumers.  N > 1 (one rank per GPU): still one logical producer -- every
rank collates its B/N rows of each batch and the collate kernel stores them
straight into the same slot of every rank's ring over NVLink (sharded ingest
+ the all-gather fused into the producing kernel); each GPU's
4 consumers get every whole batch (weak scaling in delivered samples: the
consumer count grows with N).  Test hook: TSB_BENCH_SAME_DEVICE=1 +
TSB_BENCH_BACKEND=gloo put every rank on cuda:0 (peers = IPC allocations on
one GPU) so the N > 1 path runs on a one-GPU box.

value: delivered samples/s summed over all consumers (the reference's
aggregate metric, bs/harness.py:574 + bs/cli.py:220-236), inputs resident in
HBM, native producer loop, device-timed (CUDA events), max over ranks.
e2e:   the same metric through the public API (TensorProducer(CollateLoader)
+ SharedLoader consumer processes), samples read from a PINNED HOST store by
the kernel over PCIe every step; each consumer reads back one element per
batch (.item(), the "step result"); consumer-side fetch timestamps with the
reference formula.
--impl reference: the CPU oracle port (oracle/, C + OpenMP, the reference
path restated: shuffle + collate(+augment) + CRC per batch) on the host cores.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

H, W, C = 224, 224, 3
SAMPLE_BYTES = H * W * C           # 150,528 B u8 HWC
B = 256
N_SAMPLES = 16384                  # samples_per_epoch
N_CONSUMERS = 4
RING_SLOTS = int(os.environ.get("TSB_BENCH_SLOTS", "8"))  # A/B knob
PAD = 16
OUT_BYTES = C * H * W * 4          # f32 NCHW per sample
ALG_BYTES_PER_SAMPLE = SAMPLE_BYTES + OUT_BYTES  # 752,640 B read + write (collate)
METRIC = "delivered samples/sec (all consumers)"
REF_BUDGET_S = 90.0  # reference arm: total CPU seconds the timed + warm-up steps may take
# e2e API leg: a fixed window of batches, independent of --steps
# (TSB_BENCH_E2E_BATCHES shortens it for profiler runs only)
E2E_BATCHES = int(os.environ.get("TSB_BENCH_E2E_BATCHES", 4096))
E2E_WARMUP = 64     # e2e batches before the window (consumer start-up skew)
E2E_BUFFER_DEPTH = RING_SLOTS - 2  # flow gate of the e2e producer (reference default is 2)
CHECKSUM = True     # per-batch CRC-32 in the timed producer (--checksum)
PERSIST = True      # checksum on, N=1: one persistent launch per epoch chunk (--persistent)
HOLD_S = 0.004      # value leg: the stream is held while the first batches are enqueued
NVLINK_GBS = 770.0  # measured peer copy per direction per GPU (B200_PROFILING.md)
WORKLOAD = ("C2: 1 producer + 4 same-GPU consumers via CUDA IPC zero copy, 224x224x3 u8 store "
            "-> ResNet-50-shaped f32 NCHW (crop pad16 + hflip from the reference RNG + ImageNet "
            "normalise), batch 256")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------- helpers ---
def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def reduce_over_ranks(x: float, op: str, backend: str) -> float:
    """max (device time of the slowest rank) or sum (whole-job throughput)
    of a per-rank number, on the process group's device."""
    import torch

    t = torch.tensor([float(x)], dtype=torch.float64,
                     device="cuda" if backend == "nccl" else "cpu")
    torch.distributed.all_reduce(t, op=(torch.distributed.ReduceOp.MAX if op == "max" else
                                        torch.distributed.ReduceOp.SUM))
    return float(t.item())


class Clocks:
    """SM clock + throttle-reason sampling during the timed region
    (B200_PROFILING.md clocks line).  NVML in a thread at 5 ms (the timed
    region can be a few hundred ms); nvidia-smi -lms 100 as the fallback."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, dev: int):
        self.dev = dev
        self.rows = []
        self._p = None
        self._nv = None
        self._stop = threading.Event()

    def start(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            self._nv = nv
            self._h = nv.nvmlDeviceGetHandleByIndex(self.dev)
            self._max = nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)
            self._t = threading.Thread(target=self._poll_nvml, daemon=True)
            self._t.start()
            return
        except Exception:  # noqa: BLE001 - fall back to nvidia-smi
            self._nv = None
        self._start_smi()

    def _poll_nvml(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                self.rows.append((sm, [n for n, a in self.REASONS if rs & getattr(nv, a)]))
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.005)

    def _start_smi(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self._p = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={q}",
                                        "--format=csv,noheader,nounits", "-lms", "100"],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except OSError:
            self._p = None

    def _read(self):
        for line in self._p.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def stop(self):
        if self._nv is not None:
            self._stop.set()
            self._t.join(1)
            if not self.rows:
                return {"sm_mhz": None, "sm_max_mhz": self._max, "reasons": ["no samples"]}
            return {"sm_mhz": statistics.median(r[0] for r in self.rows),
                    "sm_max_mhz": float(self._max),
                    "reasons": sorted({n for r in self.rows for n in r[1]}),
                    "samples": len(self.rows), "source": "nvml"}
        if self._p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self._p.terminate()
        try:
            self._p.wait(2)
        except subprocess.TimeoutExpired:
            self._p.kill()
        rows = self.rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[3:]) if v == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][1]) if rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows)}


def measured_hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(per_batch=True):
    """DRAM bytes per batch of the collate kernel from the committed ncu capture
    (persistent range launch / its batches; per_batch=False: the per-batch
    launch's figure)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        if per_batch:
            return d.get("collate_f32_b256_bytes_per_batch")
        return d.get("per_launch_kernel", {}).get("collate_f32_b256_bytes_per_launch")
    except (OSError, ValueError):
        return None


# ------------------------------------------------------- consumer workers ---
def device_consumer(dev, handle, slots, slot_bytes, max_consumers, cursor, warmup, steps, q,
                    control="-"):
    """Minimal consumer process: maps the ring over CUDA IPC, waits for each
    batch and releases it (device-counted ack); device-timed."""
    import torch

    torch.cuda.set_device(dev)
    from paper_2409_18749_b200 import dataplane as dp
    from paper_2409_18749_b200.ring import DeviceRing, consume_range

    ring = DeviceRing.import_handle(handle, slots, slot_bytes, max_consumers, control)
    s = torch.cuda.Stream()
    e0, e1 = dp.DeviceEvent(), dp.DeviceEvent()
    q.put(("ready", cursor))
    consume_range(ring, cursor, 1, warmup, stream=s)
    consume_range(ring, cursor, warmup + 1, steps, events=[e0, e1], stream=s)
    s.synchronize()
    q.put(("done", cursor, e0.elapsed_ms(e1)))
    ring.close()


def host_consumer(dev, handle, control, slots, slot_bytes, max_consumers, cursor, warmup, steps,
                  q, writers=1):
    """The reference consumer (bs/cli.py:252-258: map, ack, never read the
    payload): maps the ring over CUDA IPC; waits and releases through the
    host-shared control block, so it never touches its GPU channel."""
    import torch

    torch.cuda.set_device(dev)
    from paper_2409_18749_b200.ring import DeviceRing

    ring = DeviceRing.import_handle(handle, slots, slot_bytes, max_consumers, control, writers)
    q.put(("ready", cursor))
    ring.host_consume_range(cursor, 1, warmup, timestamps=False)
    times = ring.host_consume_range(cursor, warmup + 1, steps)  # native wait -> stamp -> ack
    rate = (len(times) - 1) / (times[-1] - times[0]) * B if len(times) > 1 else 0.0
    q.put(("done", cursor, rate))
    ring.close()


def api_consumer(dev, bcast, agg, cid, warmup, steps, q):
    """e2e consumer through the public API: SharedLoader over CUDA IPC; reads
    one element per batch back to the host (the step result).  Reports the
    fetch time of every batch after the warm-up."""
    import torch

    torch.cuda.set_device(dev)
    from paper_2409_18749_b200 import SharedLoader

    loader = SharedLoader(bcast, agg, consumer_id=cid)
    times, n = [], 0
    q.put(("ready", cid))
    for _epoch in range(1 << 20):
        for inp, tgt in loader:
            _ = float(inp.view(-1)[0].item())  # D2H of the step result (4 B)
            n += 1
            if n > warmup:
                times.append(time.monotonic())
            if n >= warmup + steps:
                break
        if n >= warmup + steps or loader.finished:
            break
    loader.close()
    rate = (len(times) - 1) / (times[-1] - times[0]) * B if len(times) > 1 else 0.0
    q.put(("done", cid, rate, n, times))


def common_window_rate(stamps: dict) -> tuple[float, float, int]:
    """Aggregate delivered samples/s over the window every consumer was
    streaming in: [latest first fetch, earliest last fetch]; each consumer's
    fetches inside it, by the reference formula's spirit (bs/cli.py:220-236:
    batches x batch / elapsed), summed (bs/harness.py:574).  Returns (rate,
    window seconds, batches counted)."""
    lo = max(t[0] for t in stamps.values())
    hi = min(t[-1] for t in stamps.values())
    if hi <= lo:
        return 0.0, 0.0, 0
    n = 0
    for t in stamps.values():
        n += sum(1 for x in t if lo < x <= hi)
    return n * B / (hi - lo), hi - lo, n


# --------------------------------------------------------------- ours ------
def run_ours(args):
    import multiprocessing as mp

    import numpy as np
    import torch

    rank, world, local = dist_env()
    dev = 0 if os.environ.get("TSB_BENCH_SAME_DEVICE") == "1" else local
    torch.cuda.set_device(dev)
    backend = os.environ.get("TSB_BENCH_BACKEND", "nccl")
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    from paper_2409_18749_b200 import (AugmentSpec, CollateLoader, DatasetSpec, StoreSource,
                                       TensorProducer)
    from paper_2409_18749_b200 import dataplane as dp
    from paper_2409_18749_b200._lib import GATE_HOST
    from paper_2409_18749_b200._lib import ProduceArgs
    from paper_2409_18749_b200.ring import (DeviceRing, produce_group, produce_range,
                                            restage_collate)

    K, Wm = args.steps, args.warmup
    ctx = mp.get_context("spawn")

    # ---- device-resident run (value) ----
    # One logical producer.  N = 1 is exactly C2.  At N GPUs (default
    # TSB_BENCH_FANOUT=inputs, two-stage): every rank gathers its 1/N rows of
    # each batch (compact u8) into the same slot of every rank's INPUT ring
    # (own HBM + peers over NVLink, tsb_produce_group), then each rank
    # collates the whole staged batch locally into its output ring
    # (tsb_restage_collate) -- 1x the input crosses NVLink instead of the 4x
    # larger f32 output.  TSB_BENCH_FANOUT=outputs: the collate kernel itself
    # stores its 1/N output rows into every rank's output ring (fused
    # all-gather of the outputs).  Each rank's 4 consumers see every batch.
    fanout = os.environ.get("TSB_BENCH_FANOUT", "inputs") if world > 1 else "none"
    store = StoreSource.synthetic(0, N_SAMPLES, (H, W, C), location="hbm")
    ds = DatasetSpec(store, N_SAMPLES, B, shuffle_seed=0)
    loader = CollateLoader(ds, AugmentSpec(pad=PAD, flip=True, out_dtype="float32"))
    out_writers = world if fanout == "outputs" else 1
    ring = DeviceRing(RING_SLOTS, loader.batch_nbytes, N_CONSUMERS, device=dev, control="host",
                      writers=out_writers)
    handle = ring.export()
    rings = [ring]
    in_ring, in_rings, gather_ld, tables = None, None, None, None
    if world > 1:
        from paper_2409_18749_b200 import group

        if fanout == "outputs":
            rings = group.open_group(ring, group.exchange(group.describe(ring, rank)), rank)
        else:
            from paper_2409_18749_b200.collate import _Ingest

            gather_ld = CollateLoader(ds)  # u8 rows + target indices (stage 1)
            in_ring = DeviceRing(4, gather_ld.batch_nbytes, 1, device=dev, control="host",
                                 writers=world)
            in_ring.set_cursor(0, 0)
            in_rings = group.open_group(in_ring, group.exchange(group.describe(in_ring, rank)),
                                        rank)
            tables = _Ingest(dev, B, SAMPLE_BYTES)
    q = ctx.Queue()
    procs = [ctx.Process(target=host_consumer,
                         args=(dev, handle, ring.control_name, RING_SLOTS, loader.batch_nbytes,
                               N_CONSUMERS, k, Wm, K, q, out_writers))
             for k in range(N_CONSUMERS)]
    for p in procs:
        p.start()
    for _ in procs:
        assert q.get(timeout=300)[0] == "ready"
    stream = torch.cuda.Stream()
    live = list(range(N_CONSUMERS))
    L = len(loader)
    # the reference checksums every segment it creates (bs/payload.py:218): the
    # per-batch CRC-32 (input + target) is fused into the collate kernel and
    # lands in d_crc[slot] before the slot is published
    # (N > 1: the two-stage path's local collate computes it too; the fused
    # output all-gather, fanout "outputs", runs without it)
    d_crc = (torch.zeros(RING_SLOTS, dtype=torch.int32, device=f"cuda:{dev}")
             if CHECKSUM and (world == 1 or fanout == "inputs") else None)

    def chunks(seq0, n):
        done = 0
        while done < n:
            q0 = seq0 + done
            epoch, bi = divmod(q0 - 1, L)
            m = min(n - done, L - bi)
            yield q0, epoch, bi, m
            done += m

    def stage1(seq0, n, s1):
        for q0, epoch, bi, m in chunks(seq0, n):
            produce_group(in_rings, rank, gather_ld.produce_args(epoch), rank, world, q0, bi, m,
                          [[0]] * world, stream=s1)

    def produce(seq0, n):
        """Enqueue n batches starting at global seq0 (1-based), across epochs."""
        feeder = None
        if fanout == "inputs":  # stage 1 runs beside stage 2 on its own thread + stream
            s1 = torch.cuda.Stream()
            feeder = threading.Thread(target=stage1, args=(seq0, n, s1))
            feeder.start()
        for q0, epoch, bi, m in chunks(seq0, n):
            a = loader.produce_args(epoch, with_crc=d_crc)
            a.gate = GATE_HOST  # gate on the host-shared cursors; PDL-chained kernels
            # persistent: the fused collate + CRC runs the whole chunk in one
            # cooperative launch, the slot gate on the device
            a.persistent = int(PERSIST and d_crc is not None and world == 1)
            if world == 1:
                produce_range(ring, a, q0, bi, m, live, stream=stream)
            elif fanout == "outputs":
                produce_group(rings, rank, a, rank, world, q0, bi, m, [live] * world,
                              stream=stream)
            else:
                a2 = ProduceArgs.from_buffer_copy(a)
                a2._keep = getattr(a, "_keep", None)
                a2.ingest = tables.handle
                restage_collate(in_ring, 0, ring, a2, q0, m, live, stream=stream)
        if feeder is not None:
            feeder.join()

    produce(1, Wm)
    stream.synchronize()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    t0, t1 = dp.DeviceEvent(), dp.DeviceEvent()
    # The stream is held on a host-released word while the host enqueues the
    # first batches (up to the ring depth, then the slot gate blocks it), so
    # t0 marks the device starting batch Wm+1, not the host's launch latency;
    # after the release the host keeps enqueueing ahead of the device.
    hold = DeviceRing(1, 64, 1, device=dev, control="host")
    hold.wait_free([0], 1, stream)
    t0.record(stream)
    release = threading.Timer(HOLD_S, hold.host_ack, args=(0, 1))
    clocks = Clocks(dev)
    clocks.start()
    release.start()
    produce(Wm + 1, K)
    t1.record(stream)
    stream.synchronize()
    clk = clocks.stop()
    release.join()
    torch.cuda.synchronize()
    ms = t0.elapsed_ms(t1)
    hold.close()
    parity = check_ring_parity(ring, loader, Wm + K, dp, d_crc) if world == 1 else None
    bf16 = bf16_line(dev, store, ds, K, Wm) if world == 1 else None
    consumer_rates = {}
    for _ in procs:
        msg = q.get(timeout=300)
        consumer_rates[msg[1]] = msg[2]
    for p in procs:
        p.join(60)
    # the producer stream carries only the K collate launches (gate on the host,
    # publish fused into the kernel, consecutive launches PDL-chained), so the
    # kernel's average launch duration is the timed region / K
    avg_launch_ms = ms / K
    persistent = bool(PERSIST and d_crc is not None and world == 1)
    launches = sum(1 for _ in chunks(Wm + 1, K)) if persistent else K
    if world > 1:
        ms_max = reduce_over_ranks(ms, "max", backend)
        torch.distributed.barrier()  # peers are done writing into our ring
    else:
        ms_max = ms
    value = world * N_CONSUMERS * B * K / (ms_max / 1e3)
    for r in rings + (in_rings or []):
        if r is not ring and r is not in_ring:
            r.close()
    if in_ring is not None:
        in_ring.close()
    ring.close()
    del store, loader
    if parity is not None and not parity["ok"]:
        log("PARITY FAILURE:", json.dumps(parity))

    # ---- e2e through the public API (pinned host store, PCIe ingest) ----
    e2e = run_e2e(args, ctx, dev, rank, world)

    peak, peak_src = measured_hbm_peak()
    if world == 1:
        achieved = B * ALG_BYTES_PER_SAMPLE / (avg_launch_ms / 1e3) / 1e9
        roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                    "frac": round(achieved / peak, 4),
                    "traffic": ncu_traffic(persistent) if d_crc is not None else None,
                    "traffic_per": "batch (ncu dram read + write of one launch / its batches)",
                    # the measured peak is a best-of-10 torch copy; the HGX spec figure
                    # (B200_PROFILING.md) for comparison
                    "spec_peak_gbs": 7700.0, "frac_of_spec": round(achieved / 7700.0, 4),
                    "kernel": ("collate_crc_range_kernel<f32,C=3> (persistent: collate + fused "
                               "batch CRC-32, one launch per epoch chunk)" if persistent else
                               "collate_crc_kernel<f32,C=3> (collate + fused batch CRC-32)"
                               if d_crc is not None else "collate_augment_kernel<f32,C=3>"),
                    # achieved = algorithmic bytes / device time, per batch (a
                    # persistent launch covers K / launches batches)
                    "alg_bytes_per_launch": B * ALG_BYTES_PER_SAMPLE * K // launches,
                    "avg_launch_ms": round(ms / launches, 5),
                    "batches_per_launch": round(K / launches, 2),
                    "alg_bytes_per_batch": B * ALG_BYTES_PER_SAMPLE,
                    "avg_batch_ms": round(avg_launch_ms, 5), "peak_source": peak_src}
    else:
        # binding link: each rank's NVLink egress -- its 1/N rows stored into the
        # N-1 peers' rings (u8 input rows for the two-stage path, f32 outputs else)
        row_bytes = SAMPLE_BYTES if fanout == "inputs" else OUT_BYTES
        egress = (B // world) * row_bytes * (world - 1)
        achieved = egress / (ms_max / K / 1e3) / 1e9
        roofline = {"bound": "nvlink", "achieved": round(achieved, 1), "peak": NVLINK_GBS,
                    "unit": "GB/s", "frac": round(achieved / NVLINK_GBS, 4), "traffic": None,
                    "kernel": ("passthrough_multi_kernel (u8 row all-gather) + local "
                               "collate_augment_kernel<f32>" if fanout == "inputs" else
                               "collate_augment_kernel<f32,C=3,MULTI> (fused all-gather)"),
                    "alg_bytes_per_launch": egress, "avg_launch_ms": round(ms_max / K, 5),
                    "peak_source": "B200_PROFILING.md measured peer copy, per direction per GPU",
                    "fanout": fanout,
                    **({"note": "TSB_BENCH_SAME_DEVICE test mode: every rank on one GPU, no "
                                "NVLink traffic; frac is not a link utilisation"}
                       if os.environ.get("TSB_BENCH_SAME_DEVICE") else {}),
                    "hbm_achieved_gbs": round(
                        B * ALG_BYTES_PER_SAMPLE / (ms_max / K / 1e3) / 1e9, 1)}
    result = {
        "metric": METRIC, "value": round(value, 1), "unit": "samples/s", "n_gpus": world,
        "steps": K, "warmup": Wm, "ms_per_step": round(ms_max / K, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic: SplitMix64 DirectorySource-equivalent store (reference RNG), "
                "reference Fisher-Yates epoch order",
        "config": {"workload": WORKLOAD, "global_batch": B, "batch_per_gpu": B,
                   "consumers_per_gpu": N_CONSUMERS, "samples_per_epoch": N_SAMPLES,
                   "ring_slots": RING_SLOTS, "sample": "224x224x3 u8 -> 3x224x224 f32",
                   "store": "HBM-resident (value) / pinned host (e2e)",
                   "l2": "inputs larger than L2: 2.47 GB store, 1.2 GB ring of 8 slots",
                   "parallelism": (
                       (f"two-stage: every rank gathers B/{world} u8 rows of each batch into "
                        "every rank's input ring (P2P stores over NVLink), then collates the "
                        "whole batch locally; 4 IPC consumers per GPU")
                       if fanout == "inputs" else
                       (f"sharded ingest over {world} GPUs (each collates B/{world} rows of "
                        "every batch) + all-gather fused into the collate kernel (P2P stores "
                        "into every rank's ring slot); 4 IPC consumers per GPU")
                       if world > 1 else "1 producer, 4 IPC consumers"),
                   "sync": (("persistent fused kernel: the slot-reuse gate runs on the device "
                             "against the host-shared release cursors (CTA 0 polls them and "
                             "raises a gate word) and the slot's previous publish; fused publish "
                             "(release store from the batch's completing CTA)"
                             if persistent else
                             "slot-reuse gate on the host-shared release cursors (producer "
                             "thread blocks, never the stream); fused publish (release store "
                             "from the kernel's last CTA); consecutive batches chained with "
                             "programmatic dependent launch")
                            + "; consumers: host wait + host ack (map-and-ack, "
                              "bs/cli.py:252-258)"),
                   "checksum": ("CRC-32 of every batch (input + target, as create_segment, "
                                "bs/payload.py:218), fused into the collate kernel, in the timed "
                                "region" if d_crc is not None else "off")},
        "roofline": roofline,
        "e2e": e2e,
        # per step: the collate (N=1, outputs fan-out); the row gather + the
        # collate (two-stage)
        "gpu_launches": launches if fanout != "inputs" else 2 * K,
        "clocks": clk,
        "extra": {"producer_ms": round(ms, 3),
                  "consumer_rates_samples_s": {str(k): round(v, 1) for k, v in consumer_rates.items()},
                  "produced_samples_per_s": round(B * K / (ms_max / 1e3), 1),
                  "timing": f"device events on the producer stream; the stream is held for "
                            f"{HOLD_S * 1e3:.0f} ms on a host-released word while the first "
                            f"batches are enqueued (t0 = device start of batch {Wm + 1})",
                  **({"parity": parity} if parity is not None else {}),
                  **({"bf16": bf16} if bf16 is not None else {})},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(seconds=args.cpu_seconds)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    if rank == 0:
        print(json.dumps(result), flush=True)


def oracle_batch_crc(o, epoch: int, bi: int, out_kind: int, nthreads: int) -> int:
    """CRC-32 the reference path gives batch (epoch, bi) of the C2 stream:
    oracle collate+augment of the samples order[bi*B:(bi+1)*B] (a store
    sample i = fill(derive_key(0, 0, i)), pipeline.py:139-155), followed by
    the int64 target indices (the pair payload, sl/abi.py:291-308)."""
    import numpy as np

    order = o.epoch_order(N_SAMPLES, 0, epoch)
    idx = np.ascontiguousarray(order[bi * B:(bi + 1) * B])
    mini = o.prepare_synthetic(0, 0, idx, SAMPLE_BYTES, nthreads)  # just those samples
    params = o.aug_params(0, epoch, idx, PAD)
    scale, bias = o.norm_consts()
    out = o.collate_augment(mini, np.arange(B, dtype=np.int64), H, W, C, PAD, True, 0, epoch,
                            out_kind, scale, bias, params=params, nthreads=nthreads)
    return o.crc32(idx.astype(np.int64), o.crc32(out))


def check_ring_parity(ring, loader, last_seq: int, dp, d_crc=None) -> dict:
    """After the timed region: the device CRC-32 of every batch still in the
    ring (the last `slots` produced) against the oracle's CRC of the same
    batch (a CRC gate on every run), and the checksum the
    producer computed for it (fused into the collate) against both."""
    import torch

    from oracle import oracle as o

    nthreads = os.cpu_count() or 1
    L = len(loader)
    crc = torch.zeros(1, dtype=torch.int32, device=f"cuda:{ring.device}")
    rows, ok = [], True
    for q in range(max(1, last_seq - ring.slots + 1), last_seq + 1):
        slot = ring.slot_of(q)
        epoch, bi = divmod(q - 1, L)
        dp.crc32(ring.slot_ptr(slot), loader.batch_nbytes, crc)
        torch.cuda.synchronize()
        got = int(crc.item()) & 0xFFFFFFFF
        want = oracle_batch_crc(o, epoch, bi, o.OUT_F32, nthreads)
        ready = ring.read_ready(slot)
        ok = ok and got == want and ready == q
        row = {"seq": q, "epoch": epoch, "batch": bi, "crc": f"{got:#010x}",
               "oracle": f"{want:#010x}"}
        if d_crc is not None:
            prod = int(d_crc[slot].item()) & 0xFFFFFFFF
            ok = ok and prod == want
            row["producer_crc"] = f"{prod:#010x}"
        rows.append(row)
    return {"ok": ok, "batches_checked": len(rows), "bytes_per_batch": loader.batch_nbytes,
            "how": "device CRC-32 (tsb_crc32) of each resident ring slot = f32 NCHW input + "
                   "int64 targets, vs the oracle's collate+augment of the same batch; "
                   "producer_crc = the checksum the timed producer computed (fused)",
            "batches": rows}


def bf16_line(dev, store, ds, K: int, Wm: int) -> dict:
    """C2/C3's bf16 output through the same native loop (no consumers: the
    collate alone, PDL-chained, device-timed), plus its parity on the last batch."""
    import torch

    from oracle import oracle as o
    from paper_2409_18749_b200 import AugmentSpec, CollateLoader
    from paper_2409_18749_b200 import dataplane as dp
    from paper_2409_18749_b200._lib import GATE_HOST
    from paper_2409_18749_b200.ring import DeviceRing, produce_range

    ld = CollateLoader(ds, AugmentSpec(pad=PAD, flip=True, out_dtype="bfloat16"))
    ring = DeviceRing(RING_SLOTS, ld.batch_nbytes, 1, device=dev, control="host")
    st = torch.cuda.Stream()
    L = len(ld)
    d_crc = torch.zeros(RING_SLOTS, dtype=torch.int32, device=f"cuda:{dev}") if CHECKSUM else None

    def run(seq0, n):
        done = 0
        while done < n:
            q0 = seq0 + done
            epoch, bi = divmod(q0 - 1, L)
            m = min(n - done, L - bi)
            a = ld.produce_args(epoch, with_crc=d_crc)
            a.gate = GATE_HOST
            a.persistent = int(PERSIST and d_crc is not None)
            produce_range(ring, a, q0, bi, m, [], stream=st)
            done += m

    run(1, Wm)
    st.synchronize()
    hold = DeviceRing(1, 64, 1, device=dev, control="host")
    hold.wait_free([0], 1, st)
    e0, e1 = dp.DeviceEvent(), dp.DeviceEvent()
    e0.record(st)
    rel = threading.Timer(HOLD_S, hold.host_ack, args=(0, 1))
    rel.start()
    run(Wm + 1, K)
    e1.record(st)
    st.synchronize()
    rel.join()
    ms = e0.elapsed_ms(e1)
    hold.close()
    last = Wm + K
    epoch, bi = divmod(last - 1, L)
    crc = torch.zeros(1, dtype=torch.int32, device=f"cuda:{dev}")
    dp.crc32(ring.slot_ptr(ring.slot_of(last)), ld.batch_nbytes, crc, st)
    st.synchronize()
    got = int(crc.item()) & 0xFFFFFFFF
    want = oracle_batch_crc(o, epoch, bi, o.OUT_BF16, os.cpu_count() or 1)
    prod = (int(d_crc[ring.slot_of(last)].item()) & 0xFFFFFFFF) if d_crc is not None else None
    ring.close()
    alg = B * (SAMPLE_BYTES + C * H * W * 2)
    peak, _ = measured_hbm_peak()
    achieved = alg / (ms / K / 1e3) / 1e9
    return {"kernel": ("collate_crc_range_kernel<bf16,C=3> (persistent, fused batch CRC-32)"
                       if PERSIST and d_crc is not None else
                       "collate_crc_kernel<bf16,C=3> (collate + fused batch CRC-32)"
                       if d_crc is not None else "collate_augment_kernel<bf16,C=3>"),
            "avg_launch_ms": round(ms / K, 5),
            "delivered_samples_s": round(N_CONSUMERS * B * K / (ms / 1e3), 1),
            "achieved_gbs": round(achieved, 1), "frac": round(achieved / peak, 4),
            "alg_bytes_per_launch": alg,
            "parity": {"ok": got == want and prod in (None, want), "crc": f"{got:#010x}",
                       "oracle": f"{want:#010x}", "seq": last,
                       **({"producer_crc": f"{prod:#010x}"} if prod is not None else {})}}


def run_e2e(args, ctx, dev, rank, world):
    """e2e through the public API.  N = 1: TensorProducer over a pinned-host
    store (gather-kernel ingest) and 4 SharedLoader processes.  N > 1: rank 0
    runs ONE TensorProducer(devices=[every rank's GPU]) -- each GPU ingests
    its 1/N rows of every batch over its own PCIe link and the collate kernel
    stores them into every GPU's ring (fused all-gather) -- and every rank
    runs 4 SharedLoader(device=its GPU) consumers."""
    import torch

    from paper_2409_18749_b200 import (AugmentSpec, CollateLoader, DatasetSpec, StoreSource,
                                       TensorProducer)

    K, Wm = args.steps, args.warmup
    tmp = f"/tmp/tsb-bench-{os.getpid()}"
    if world > 1:  # one endpoint pair for the whole job, created by rank 0
        obj = [tmp]
        torch.distributed.broadcast_object_list(obj, src=0)
        tmp = obj[0]
        devs = [None] * world
        torch.distributed.all_gather_object(devs, dev)
    os.makedirs(tmp, exist_ok=True)
    bcast, agg = f"unix:{tmp}/b.sock", f"unix:{tmp}/a.sock"
    producer = None
    if rank == 0:
        store = StoreSource.synthetic(0, N_SAMPLES, (H, W, C), location="pinned")
        ds = DatasetSpec(store, N_SAMPLES, B, shuffle_seed=0)
        loader = CollateLoader(ds, AugmentSpec(pad=PAD, flip=True, out_dtype="float32"))
        # N > 1: the same fan-out design as the device-timed value (two-stage
        # input all-gather by default, TSB_BENCH_FANOUT=outputs for the fused one)
        fan = "inputs" if os.environ.get("TSB_BENCH_FANOUT", "inputs") == "inputs" else "sharded"
        producer = TensorProducer(loader, bcast, agg, buffer_depth=E2E_BUFFER_DEPTH,
                                  min_consumers=N_CONSUMERS * world,
                                  ring_slots=RING_SLOTS, heartbeat_timeout_s=60.0,
                                  devices=devs if world > 1 else None, fanout=fan)
        producer._start()  # listeners up before any rank's consumers dial
    if world > 1:
        torch.distributed.barrier()
    q = ctx.Queue()
    # a fixed window independent of --steps (start-up skew of a few batches
    # must not decide the number)
    Wm, K = E2E_WARMUP, max(K, E2E_BATCHES)
    procs = [ctx.Process(target=api_consumer,
                         args=(dev, bcast, agg, 1000 + 100 * rank + k, Wm, K, q))
             for k in range(N_CONSUMERS)]
    for p in procs:
        p.start()
    total = Wm + K
    t_start = time.monotonic()
    produced = 0
    if producer is not None:
        while produced < total:
            for _ in producer:
                produced += 1
                if produced >= total:
                    break
        producer.join(drain_timeout_s=60)
    h2d = B * SAMPLE_BYTES  # every sample row (sharded multi-GPU ingest)
    if producer is not None and world == 1 and loader._ingest is not None and produced:
        # the ingest counts what it enqueued: the rows the crop reads,
        # plus the index and parameter uploads
        h2d = int(round(loader._ingest.bytes_enqueued() / produced))
    rates, stamps = {}, {}
    for _ in procs:
        msg = q.get(timeout=600)
        while msg[0] != "done":
            msg = q.get(timeout=600)
        rates[msg[1]] = msg[2]
        stamps[msg[1]] = msg[4]
    for p in procs:
        p.join(60)
    if world > 1:
        torch.distributed.barrier()  # every consumer is done before the rings go
    drift = None
    if producer is not None:
        drift = producer._ledger.drift_max
        producer.close()
    wall = time.monotonic() - t_start
    value, window_s, counted = common_window_rate(stamps)
    if world > 1:
        value = reduce_over_ranks(value, "sum", os.environ.get("TSB_BENCH_BACKEND", "nccl"))
    per = list(rates.values())
    spread = (max(per) - min(per)) / max(per) if per and max(per) > 0 else None
    path = ("TensorProducer(CollateLoader(pinned-host StoreSource)) -> 4 SharedLoader processes "
            "(CUDA IPC); each batch's sample rows that the crop reads cross PCIe by the copy "
            "engine, with the host-derived crop/flip table; consumers .item() one element per "
            "batch")
    if world > 1:
        path = (f"one TensorProducer(devices={world} GPUs, fanout="
                f"{'inputs' if os.environ.get('TSB_BENCH_FANOUT', 'inputs') == 'inputs' else 'sharded'}"
                ": each GPU reads its 1/N rows of every batch from pinned host memory and stores "
                "them into every GPU's ring) -> 4 SharedLoader(device=g) processes per GPU; "
                "consumers .item() per batch")
    return {"value": round(value, 1), "unit": "samples/s",
            "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": 4 * N_CONSUMERS * world,
            "path": path,
            "window": {"batches_per_consumer": K, "warmup_batches": Wm,
                       "seconds": round(window_s, 3), "batches_counted": counted,
                       "how": "aggregate over the interval every consumer was fetching in "
                              "(latest first fetch to earliest last fetch)"},
            "per_consumer": {str(k): round(v, 1) for k, v in rates.items()},
            "per_consumer_spread": None if spread is None else round(spread, 4),
            "sum_per_consumer": round(sum(per), 1),
            "buffer_depth": E2E_BUFFER_DEPTH, "ledger_drift_max": drift,
            "checksum": "device CRC-32 of every batch in its Announce (TensorProducer default, "
                        "as the reference's create_segment, bs/payload.py:218)",
            "wall_s": round(wall, 2), "batches_produced": produced}


# -------------------------------------------------------------- CPU port ----
def cpu_reference_step(o, store, order, bi, nthreads, out, scale, bias):
    """One batch of the reference CPU path, restated (oracle/): collate +
    augment (f32 NCHW) on all threads, then the segment CRC (payload.py:218)."""
    idx = order[bi * B:(bi + 1) * B]
    o.collate_augment(store, idx, H, W, C, PAD, True, 0, 0, o.OUT_F32, scale, bias,
                      nthreads=nthreads, out=out)
    return o.crc32(out)


def reference_unmodified(timeout_s: float = 300.0):
    """The UNMODIFIED reference (baseline/_ref, batchsocket run_scenario in
    shared mode, tools/ref_cpu_bench.py) at C2's shape: 4 consumers, B=256,
    224x224x3 u8 -- it has no augment, so its batch is the collated u8 bytes
    (SURVEY.md §8a A6).  None when the install is absent."""
    cmd = [sys.executable, os.path.join(ROOT, "tools", "ref_cpu_bench.py"), "--only", "c2",
           "--epoch-len", "30"]
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout_s, cwd=ROOT)
        line = [x for x in r.stdout.splitlines() if x.startswith("{")][-1]
        d = json.loads(line)
    except (subprocess.SubprocessError, IndexError, ValueError, OSError) as exc:
        return {"unavailable": f"{type(exc).__name__}: {exc}"[:200]}
    if "unavailable" in d:
        return d
    return {"value": d["aggregate_samples_s"], "unit": "samples/s", "cores": d["workers"],
            "kind": "reference",
            "sample": f"unmodified reference (baseline/_ref) run_scenario shared mode: "
                      f"{d['consumers']} consumers, B={d['batch_size']}, 224x224x3 u8 (no "
                      f"augment exists in the reference), {d['epochs']} epochs x "
                      f"{d['epoch_len']} batches, workers={d['workers']}, "
                      f"wall {d['wall_s']} s",
            "per_consumer": d["per_consumer_samples_s"], "cpu_model": d.get("cpu")}


def cpu_baseline(seconds: float = 15.0):
    from oracle import oracle as o

    nthreads = os.cpu_count() or 1
    n_store = N_SAMPLES
    store = o.make_store(0, n_store, SAMPLE_BYTES, nthreads=nthreads)
    order = o.epoch_order(n_store, 0, 0)
    scale, bias = o.norm_consts()
    import numpy as np

    out = np.empty((B, C, H, W), dtype=np.float32)
    cpu_reference_step(o, store, order, 0, nthreads, out, scale, bias)  # warm
    t0 = time.monotonic()
    n = 0
    while True:
        cpu_reference_step(o, store, order, n % (n_store // B), nthreads, out, scale, bias)
        n += 1
        if time.monotonic() - t0 >= seconds or n >= 200:
            break
    dt = time.monotonic() - t0
    produced = n * B / dt
    # the same step on one thread (the CPU augment oracle on
    # 1 thread and on nproc threads), a few batches
    t1, n1 = time.monotonic(), 0
    while n1 < 1 or (time.monotonic() - t1 < min(3.0, seconds / 5) and n1 < 20):
        cpu_reference_step(o, store, order, n1 % (n_store // B), 1, out, scale, bias)
        n1 += 1
    produced_1t = n1 * B / (time.monotonic() - t1)
    return {"value": round(produced * N_CONSUMERS, 1), "unit": "samples/s", "cores": nthreads,
            "single_thread_produced_samples_per_s": round(produced_1t, 1),
            "kind": "port",
            "sample": f"{n} batches x {B} samples ({dt:.1f} s): oracle C/OpenMP collate+augment "
                      f"f32 NCHW + CRC-32 per batch, {nthreads} threads; delivered = "
                      f"{N_CONSUMERS} zero-copy consumers x produced",
            "produced_samples_per_s": round(produced, 1), "cpu_model": _cpu_model(),
            "same_config": True, "samples_per_epoch": n_store,
            "reference": reference_unmodified()}


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle as o

    import numpy as np

    nthreads = os.cpu_count() or 1
    n_store = N_SAMPLES  # the same store as the GPU arm (same_config)
    store = o.make_store(0, n_store, SAMPLE_BYTES, nthreads=nthreads)
    order = o.epoch_order(n_store, 0, 0)
    scale, bias = o.norm_consts()
    out = np.empty((B, C, H, W), dtype=np.float32)
    # each step = a bounded sample of the C2 batch: the whole batch when the run
    # fits in ~REF_BUDGET_S, else the first `b` rows (same per-sample work), so
    # `--steps K --warmup W` with the driver's K still ends within minutes
    t1 = time.monotonic()
    cpu_reference_step(o, store, order, 0, nthreads, out, scale, bias)
    step_s = time.monotonic() - t1
    b = B
    if step_s * (args.steps + args.warmup) > REF_BUDGET_S:
        b = max(8, int(B * REF_BUDGET_S / (step_s * (args.steps + args.warmup))))
    outb = np.empty((b, C, H, W), dtype=np.float32)

    def step(i):
        bi = i % (n_store // B)
        idx = order[bi * B:bi * B + b]
        o.collate_augment(store, idx, H, W, C, PAD, True, 0, 0, o.OUT_F32, scale, bias,
                          nthreads=nthreads, out=outb)
        return o.crc32(outb)

    for i in range(args.warmup):
        step(i)
    t0 = time.monotonic()
    for i in range(args.steps):
        step(i)
    dt = time.monotonic() - t0
    value = N_CONSUMERS * b * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 1), "unit": "samples/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * dt / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (same store/order/augment as ours)",
        "config": {"workload": WORKLOAD, "global_batch": B, "samples_per_epoch": n_store,
                   "consumers_per_gpu": N_CONSUMERS, "same_config": True},
        "cpu_baseline": {"value": round(value, 1), "unit": "samples/s", "cores": nthreads,
                         "kind": "port",
                         "sample": f"{args.steps} steps x {b} samples (of a {B}-sample batch): "
                                   f"oracle C/OpenMP collate+augment f32 + CRC-32, "
                                   f"{N_CONSUMERS} zero-copy consumers",
                         "cpu_model": _cpu_model()},
        "e2e": {"value": round(value, 1), "unit": "samples/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    # a wedged multi-process run (a peer rank or consumer died) must end, not hang
    import faulthandler

    faulthandler.dump_traceback_later(float(os.environ.get("TSB_BENCH_WATCHDOG_S", 1500)),
                                      exit=True)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2048)
    ap.add_argument("--warmup", type=int, default=16)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--checksum", default="on", choices=["on", "off"],
                    help="per-batch CRC-32 in the timed producer (the reference's create_segment "
                         "checksums every segment)")
    ap.add_argument("--persistent", default="on", choices=["on", "off"],
                    help="checksum on, N=1: one persistent fused launch per epoch chunk "
                         "(off: one fused launch per batch, PDL-chained)")
    args = ap.parse_args()
    global CHECKSUM, PERSIST
    CHECKSUM = args.checksum == "on"
    PERSIST = args.persistent == "on"
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
