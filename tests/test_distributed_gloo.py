"""T6 — the multi-GPU exchange (final all-gather of change-point events) on the CPU with the
gloo backend, world sizes 2 and 4: rank 0 receives every rank's records, in global
(series, t) order, with zero padding removed; shard ranges tile the global series set."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2410_12588_b200 import bocd, distributed as D


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _records(rank, n):
    ev = np.zeros(n, dtype=bocd.EVENT_DTYPE)
    ev["series"] = rank * 1000 + np.arange(n) // 2
    ev["t"] = 10 + np.arange(n)
    ev["cp_index"] = ev["t"] - 3
    ev["flags"] = 1
    ev["p_new"] = 0.95
    return torch.from_numpy(ev.view(np.uint8).reshape(n, 40).copy())


def _worker(rank, world, port, counts, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = D.allgather_events(_records(rank, counts[rank]))
        tmax = D.max_over_ranks(float(rank) * 1.5, torch.device("cpu"))
        if rank == 0:
            q.put((D.records_to_numpy(out).tolist(), tmax))
        else:
            assert out is None
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,counts", [(2, [3, 5]), (4, [0, 4, 1, 2])])
def test_allgather_events_gloo(world, counts):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, counts, q)) for r in range(world)]
    for p in procs:
        p.start()
    got, tmax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = np.concatenate([D.records_to_numpy(_records(r, counts[r])) for r in range(world)])
    assert got == want.tolist()
    assert tmax == 1.5 * (world - 1)
    series = [g[0] for g in got]
    assert series == sorted(series)


def test_shard_ranges_tile():
    for S, W in [(32768, 8), (100000, 8), (10, 4), (3, 4)]:
        spans = [D.shard_range(S, r, W) for r in range(W)]
        assert spans[0][0] == 0 and spans[-1][1] == S
        for (a, b), (c, d) in zip(spans, spans[1:]):
            assert b == c and a <= b
