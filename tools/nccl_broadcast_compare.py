"""NCCL comparison point for the multi-GPU fan-out: the
"collate on one GPU, then ncclBroadcast" baseline the fused sharded-ingest
kernel (bench.py --gpus N, tsb_produce_group) is measured against.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/nccl_broadcast_compare.py

Per step: rank 0 collates a B=256 batch (bf16 or f32 NCHW) with the same
fused kernel, then NCCL broadcasts it to every rank; also ncclAllGather of
sharded collates (each rank collates B/N rows, then all-gathers).  Device
time, max over ranks; rank 0 prints one JSON line.
"""

from __future__ import annotations

import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2409_18749_b200 import AugmentSpec, CollateLoader, DatasetSpec, StoreSource

    dtype = os.environ.get("TSB_DTYPE", "bfloat16")
    steps, warm = int(os.environ.get("TSB_STEPS", 64)), 8
    N, B = 16384, 256
    store = StoreSource.synthetic(0, N, (224, 224, 3), location="hbm")
    ld = CollateLoader(DatasetSpec(store, N, B), AugmentSpec(out_dtype=dtype), with_target=False)
    buf = torch.empty(ld.batch_nbytes, dtype=torch.uint8, device="cuda")
    shard = B // world
    sample_out = ld.input_nbytes // B
    part = torch.empty(shard * sample_out, dtype=torch.uint8, device="cuda")
    _, dorder = ld.order(0)
    from paper_2409_18749_b200 import dataplane as dp

    a = ld.augment
    h, w, c = store.sample_shape

    def bcast_step(i):
        if rank == 0:
            ld.produce_into(buf.data_ptr(), 0, i % len(ld))
        dist.broadcast(buf, 0)

    def allgather_step(i):
        bi = i % len(ld)
        idx = dorder[bi * B + rank * shard: bi * B + (rank + 1) * shard]
        dp.collate_augment(store.samples, idx, shard, h, w, c, a.pad, a.flip, a.seed, 0,
                           a.out_kind, part, scale=ld._scale, bias=ld._bias)
        dist.all_gather_into_tensor(buf[:B * sample_out] if world * shard == B else buf, part)

    res = {"n_gpus": world, "dtype": dtype, "batch": B, "steps": steps}
    for name, fn in (("collate_then_ncclBroadcast", bcast_step),
                     ("sharded_collate_then_ncclAllGather", allgather_step)):
        for i in range(warm):
            fn(i)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(steps):
            fn(i)
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / steps], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        res[name] = {"ms_per_batch": round(ms, 4),
                     "delivered_samples_per_s_one_consumer_per_gpu": round(world * B / ms * 1e3, 1)}
    if rank == 0:
        print(json.dumps(res), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
