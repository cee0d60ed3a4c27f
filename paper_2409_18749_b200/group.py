"""Multi-GPU producer group: one process per GPU, one ring per GPU, sharded
ingest with the all-gather fused into the producing kernel.

Rank r of G owns the ring on its GPU.  Every rank collates rows
``shard_rows(B, r, G)`` of each batch and stores them into the same slot of
every rank's ring (its own HBM + the peers' over NVLink P2P stores), then
publishes its own ready word in each ring (``tsb_produce_group``).  The
control plane here is only the one-time exchange of ring descriptors (CUDA
IPC handle + host-shared control block name) over ``torch.distributed``;
there is no per-batch collective.
"""

from __future__ import annotations

from . import segment as sg


def shard_rows(batch_size: int, shard: int, n_shards: int) -> tuple[int, int]:
    """Rows [lo, hi) of a batch produced by `shard` (mirrors tsb_produce_group)."""
    if not 0 <= shard < n_shards or batch_size < n_shards:
        raise ValueError(f"bad shard {shard}/{n_shards} of a batch of {batch_size}")
    return shard * batch_size // n_shards, (shard + 1) * batch_size // n_shards


def exchange(desc: sg.RingDescriptor, group=None) -> list[sg.RingDescriptor]:
    """All ranks' ring descriptors, in rank order (one all_gather_object)."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    names = [None] * world
    dist.all_gather_object(names, (dist.get_rank(group), desc.name()), group=group)
    out = [None] * world
    for r, name in names:
        out[r] = sg.RingDescriptor.parse(name)
    if any(d is None for d in out):
        raise ValueError("a rank sent no ring descriptor")
    return out


def open_group(own, descs: list[sg.RingDescriptor], rank: int) -> list:
    """Ring handles of the whole group in rank order: `own` at `rank`, the
    peers' rings opened over CUDA IPC (peer GPUs: P2P mappings)."""
    from .ring import DeviceRing

    rings = []
    for r, d in enumerate(descs):
        if r == rank:
            rings.append(own)
        else:
            rings.append(DeviceRing.import_handle(d.ipc_handle, d.slots, d.slot_bytes,
                                                  d.max_consumers, d.control, d.writers))
    return rings


def describe(ring, rank: int, per_slot: int = 0, samples: int = 0) -> sg.RingDescriptor:
    import os

    return sg.RingDescriptor(rank, os.getpid(), ring.device, ring.slots, ring.slot_bytes,
                             ring.max_consumers, ring.export(), ring.control_name, ring.writers,
                             per_slot, samples)
