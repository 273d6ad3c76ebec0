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
