"""Host policy of the shared stream: admission, rubberband retention, drift.

Restates the reference's producer policy (bs/producer.py:114-269) for the
device ring.  Data-path release is device-counted (ring cursors); the host
ledger keeps the wire-level ack bookkeeping (ack-on-fetch, drift series,
exactly-once accounting) and decides which device cursors gate a slot.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import NamedTuple

from .wire import ADMIT_IMMEDIATE, ADMIT_RUBBERBAND, ADMIT_WAIT

_FRACTION_EPS = 1e-9  # producer.py:114-116


def admission_code(progress_batches: int, epoch_len: int, fraction: float) -> int:
    """producer.py:119-130: 0 progress -> immediate; strictly inside the
    rubberband window -> rubberband replay; otherwise wait for the next epoch."""
    if progress_batches == 0:
        return ADMIT_IMMEDIATE
    if progress_batches + _FRACTION_EPS < fraction * epoch_len:
        return ADMIT_RUBBERBAND
    return ADMIT_WAIT


def retention_window(fraction: float, epoch_len: int) -> int:
    """producer.py:133-135: leading batches retained for rubberband replay."""
    return math.ceil(fraction * epoch_len - _FRACTION_EPS)


def seq_of(epoch: int, index: int, epoch_len: int) -> int:
    """1-based global sequence of a batch (producer.py:99,405-406 use 0-based)."""
    return epoch * epoch_len + index + 1


def rebatch_epoch_len(samples_per_epoch: int, producer_epoch_len: int, per_slot: int,
                      batch_size: int) -> int:
    """Batches per epoch of a consumer with its own batch size: the reference's
    drop-last ``N // b`` (pipeline.py:77-79), capped by the samples the
    producer's own drop-last epoch covers (producer_epoch_len * per_slot)."""
    covered = producer_epoch_len * per_slot
    n = min(samples_per_epoch, covered) if samples_per_epoch else covered
    return n // batch_size


def window_slots(batch_size: int, per_slot: int) -> int:
    """Most producer slots one consumer batch window (starting at a multiple
    of batch_size) can touch."""
    if per_slot % batch_size == 0:
        return 1
    if batch_size % per_slot == 0:
        return batch_size // per_slot
    return -(-batch_size // per_slot) + 1


class WindowPlan(NamedTuple):
    k0: int              # first producer batch (slot) the window touches
    k1: int              # last one
    offset: int          # sample offset of the window inside batch k0
    zero_copy: bool      # inside one slot: a view, held until the next step
    release_before: int  # producer batches [0, release_before) are free before this step
    release_after: int   # gathered windows: batches [0, release_after) are free after the gather


def rebatch_window_plan(j: int, batch_size: int, per_slot: int) -> WindowPlan:
    """Batch j of a consumer with its own batch size b = stream samples
    [j*b, (j+1)*b) of the epoch order (the reference's batch for b,
    pipeline.py:113-123), laid over producer batches of per_slot samples."""
    first = j * batch_size
    k0, k1 = first // per_slot, (first + batch_size - 1) // per_slot
    return WindowPlan(k0, k1, first - k0 * per_slot, k0 == k1, k0,
                      (first + batch_size) // per_slot)


@dataclass
class ConsumerRecord:
    consumer_id: int
    cursor: int                  # device cursor index in the ring
    last_heartbeat: float
    join_epoch: int
    admitted: bool = False
    waiting_for_epoch: int | None = None
    ack_seq: int = 0             # highest wire-acked seq (1-based; 0 = none)
    conn: object = None
    bcast: object = None
    replay: list = field(default_factory=list)
    device: int = -1             # the consumer's GPU
    ring: int = 0                # index of the producer ring it maps (one per GPU)
    batch_size: int = 0          # own batch size (0 = the producer's)
    ack_epoch: int = -1          # heterogeneous consumers: producer batches acked so far
    ack_k: int = 0


class Ledger:
    """Wire-level ack ledger: which admitted consumers still owe an ack per seq."""

    def __init__(self):
        self.pending: dict[int, set] = {}
        self.drift_max = 0
        self.drift_series: list[tuple[float, int]] = []

    def add(self, seq: int, consumers) -> None:
        self.pending[seq] = set(consumers)

    def ack(self, cid: int, seq: int) -> bool:
        owed = self.pending.get(seq)
        if owed is None or cid not in owed:
            return False
        owed.discard(cid)
        if not owed:
            del self.pending[seq]
        return True

    def remove_consumer(self, cid: int) -> None:
        for seq in list(self.pending):
            self.pending[seq].discard(cid)
            if not self.pending[seq]:
                del self.pending[seq]

    def pending_count(self) -> int:
        return len(self.pending)

    def sample_drift(self, now: float, records) -> None:
        cur = [r.ack_seq for r in records if r.admitted]
        if not cur:
            return
        gap = max(cur) - min(cur)
        if gap > self.drift_max:
            self.drift_max = gap
        if not self.drift_series or self.drift_series[-1][1] != gap:
            self.drift_series.append((now, gap))
