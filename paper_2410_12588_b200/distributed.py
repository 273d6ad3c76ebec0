"""Series sharding + the one data-path exchange of a multi-GPU run.

Series are independent, so rank g of G owns a contiguous block of
global series and runs the resident kernel on it with no communication during
compute.  The only exchange is the final all-gather of the compacted
change-point events (40-byte falcon_bocd_event records that already carry
GLOBAL series ids, via falcon_bocd_config.series_base): an all_gather of the
per-rank counts, then an all_gather_into_tensor of the event records padded to
the largest count (NCCL has no all-gather-v), over NVLink / NVSwitch.  Rank 0
keeps the concatenation, which is in global (series, t) order because shards
are contiguous and each shard's drain is (series, t) ordered.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

RECORD_BYTES = 40


def shard_range(n_global: int, rank: int, world: int):
    """Contiguous block [lo, hi) of global series owned by `rank` (ceil split)."""
    per = -(-n_global // world)
    lo = min(n_global, rank * per)
    return lo, min(n_global, lo + per)


def allgather_events(records: torch.Tensor, group=None, dst: int = 0):
    """records: uint8 [n, 40] on this rank's device (NCCL) or CPU (gloo).  Returns the
    concatenated uint8 [N, 40] tensor on rank `dst` (None elsewhere)."""
    assert records.dtype == torch.uint8 and records.dim() == 2 and records.shape[1] == RECORD_BYTES
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = records.device
    n = torch.tensor([records.shape[0]], dtype=torch.int64, device=dev)
    counts = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(counts, n, group=group)
    counts = [int(c.item()) for c in counts]
    m = max(max(counts), 1)
    padded = torch.zeros((m, RECORD_BYTES), dtype=torch.uint8, device=dev)
    if records.shape[0]:
        padded[: records.shape[0]] = records
    if dist.get_backend(group) == "nccl":
        out = torch.empty((world * m, RECORD_BYTES), dtype=torch.uint8, device=dev)
        dist.all_gather_into_tensor(out, padded, group=group)
        parts = [out[r * m: r * m + counts[r]] for r in range(world)]
    else:
        bufs = [torch.empty_like(padded) for _ in range(world)]
        dist.all_gather(bufs, padded, group=group)
        parts = [bufs[r][: counts[r]] for r in range(world)]
    if rank != dst:
        return None
    return torch.cat(parts, 0)


class ShardedBocd:
    """Rank `rank`'s shard of a batched BOCD over `n_global` independent series (S:176-177:
    per-series states are single-owner; one analyzer per node).  The rank owns the
    contiguous global series [lo, hi) = shard_range(n_global, rank, world) and runs the
    device kernels on them with no communication; `gather_changepoints` is the run's one
    exchange.  A rank whose shard is empty (world > n_global) holds no batch.

    batch_factory(n_series, series_base=..., device=..., **bocd_kwargs) builds the local
    batch (default: bocd.BocdBatch; the CPU tests inject a stand-in)."""

    def __init__(self, n_global: int, rank: int | None = None, world: int | None = None,
                 device=None, batch_factory=None, group=None, **bocd_kwargs):
        if rank is None:
            rank = dist.get_rank(group) if dist.is_initialized() else 0
        if world is None:
            world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.n_global, self.rank, self.world, self.group = int(n_global), int(rank), int(world), group
        self.lo, self.hi = shard_range(self.n_global, self.rank, self.world)
        if batch_factory is None:
            from .bocd import BocdBatch as batch_factory
        self.device = device
        self.batch = (batch_factory(self.hi - self.lo, series_base=self.lo, device=device, **bocd_kwargs)
                      if self.hi > self.lo else None)

    @property
    def n_local(self) -> int:
        return self.hi - self.lo

    def update_chunk(self, x_local, **kw):
        """Absorb x_local [n_local][T] (rows = global series lo .. hi-1)."""
        if self.batch is not None:
            return self.batch.update_chunk(x_local, **kw)
        return None

    def local_changepoints(self, device_out: bool):
        """This shard's drained events as uint8 [n, 40] records and its overflow flag."""
        if self.batch is None:
            dev = torch.device("cuda", self.device) if device_out and isinstance(self.device, int) else (
                self.device if device_out else torch.device("cpu"))
            return torch.zeros((0, RECORD_BYTES), dtype=torch.uint8, device=dev), False
        recs, dropped = self.batch.changepoints(device_out=device_out)
        if not isinstance(recs, torch.Tensor):
            recs = torch.from_numpy(np.ascontiguousarray(recs).view(np.uint8).reshape(-1, RECORD_BYTES).copy())
        return recs, bool(dropped)

    def gather_changepoints(self, dst: int = 0):
        """Drain every shard and all-gather the events (NCCL: device records over NVLink; gloo:
        host records).  Returns (records uint8 [N, 40] in global (series, t) order, dropped on any
        rank) on rank `dst`, (None, dropped) elsewhere; single process: the local drain."""
        multi = dist.is_initialized() and dist.get_world_size(self.group) > 1
        nccl = multi and dist.get_backend(self.group) == "nccl"
        recs, dropped = self.local_changepoints(device_out=nccl)
        if not multi:
            return recs, dropped
        out = allgather_events(recs, group=self.group, dst=dst)
        dev = recs.device
        dropped_any = max_over_ranks(float(dropped), dev, group=self.group) > 0
        return out, dropped_any

    def close(self):
        if self.batch is not None:
            self.batch.close()
            self.batch = None


def run_sharded(x_source, n_global: int, T: int, chunk: int, device=None, batch_factory=None,
                group=None, **bocd_kwargs):
    """Whole sharded run: every rank absorbs T steps of its shard in chunks of `chunk`
    (x_source(lo, hi, t0, n) -> [hi-lo][n] observations of global series lo..hi-1, steps
    t0..t0+n-1, generated or loaded where they are used: nothing is scattered), then the
    events are all-gathered once.  Returns (events as a numpy falcon_bocd_event array in
    global (series, t) order, dropped) on rank 0, (None, dropped) on other ranks."""
    sb = ShardedBocd(n_global, device=device, batch_factory=batch_factory, group=group, **bocd_kwargs)
    try:
        if sb.n_local:
            for t0 in range(0, T, chunk):
                sb.update_chunk(x_source(sb.lo, sb.hi, t0, min(chunk, T - t0)))
        recs, dropped = sb.gather_changepoints()
    finally:
        sb.close()
    return (records_to_numpy(recs) if recs is not None else None), dropped


def gather_fixed(records: torch.Tensor, meta: torch.Tensor, group=None):
    """Stream-ordered all-gather of one drain whose size the host does not know yet: every
    rank contributes its fixed-capacity record buffer (uint8 [cap, 40]) and its drain meta
    (int64 [4], total first), both on the device, so nothing waits for the host.  Returns
    (records [world * cap, 40], metas [world * 4]) on every rank; compact_gathered() keeps
    the valid prefix of each rank's block."""
    world = dist.get_world_size(group)
    out = torch.empty((world * records.shape[0], RECORD_BYTES), dtype=torch.uint8, device=records.device)
    metas = torch.empty(world * meta.numel(), dtype=meta.dtype, device=meta.device)
    dist.all_gather_into_tensor(metas, meta.contiguous(), group=group)
    dist.all_gather_into_tensor(out, records.contiguous(), group=group)
    return out, metas


def compact_gathered(records: torch.Tensor, metas: torch.Tensor, world: int):
    """The valid events of a gather_fixed result, rank by rank (global (series, t) order)."""
    cap = records.shape[0] // world
    m = metas.view(world, -1).cpu()
    parts = [records[r * cap: r * cap + int(m[r, 0])] for r in range(world)]
    return torch.cat(parts, 0), bool(m[:, 1].any()), bool((m[:, 3] == 0).any())


def records_to_numpy(records: torch.Tensor):
    """uint8 [n, 40] records -> numpy structured array (falcon_bocd_event layout)."""
    from .bocd import EVENT_DTYPE
    raw = records.contiguous().cpu().numpy()
    return np.frombuffer(raw.tobytes(), dtype=EVENT_DTYPE) if raw.size else np.empty(0, EVENT_DTYPE)


def max_over_ranks(value: float, device, group=None) -> float:
    """Max of a per-rank scalar (timings are reported as the max over ranks)."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
