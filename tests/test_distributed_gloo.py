"""T6 — the multi-GPU exchange (final all-gather of change-point events) on the CPU with the
gloo backend, world sizes 2, 4 and 8: rank 0 receives every rank's records, in global
(series, t) order, with zero padding removed; shard ranges tile the global series set; the
package's sharded driver (distributed.run_sharded / ShardedBocd) gives every rank its
contiguous shard, feeds it its own rows only, and returns on rank 0 exactly the events a
single process over all series would report (S:176-177 per-series independence; P:692-695
one analyzer per node).  The per-rank batch is a stand-in (no GPU here) whose events are a
deterministic function of (global series, t, observation)."""
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


@pytest.mark.parametrize("world,counts", [(2, [3, 5]), (4, [0, 4, 1, 2]),
                                          (8, [2, 0, 7, 1, 1, 0, 3, 5])])
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


class _StandInBatch:
    """CPU stand-in for bocd.BocdBatch: reports an event (t, cp_index = t - 2, p_new = x)
    whenever the observation of series s at step t satisfies (s + t) % 7 == 0, and checks it is
    only ever fed its own series' rows."""

    def __init__(self, n, series_base=0, device=None, **kw):
        self.n, self.base, self.t, self.ev, self.kw = n, series_base, 0, [], kw

    def update_chunk(self, x):
        assert x.shape[0] == self.n
        for i in range(self.n):
            s = self.base + i
            for j in range(x.shape[1]):
                t = self.t + j
                assert float(x[i, j]) == _obs(s, t), "a rank was fed another shard's rows"
                if (s + t) % 7 == 0:
                    self.ev.append((s, t, t - 2, 1, 0, float(x[i, j])))
        self.t += x.shape[1]

    def changepoints(self, device_out=False):
        ev = np.array(sorted(self.ev), dtype=bocd.EVENT_DTYPE)
        self.ev = []
        return ev, False

    def close(self):
        pass


def _obs(s, t):
    return 1.0 + 0.001 * s + 1e-6 * t


def _source(lo, hi, t0, n):
    return torch.tensor([[_obs(s, t) for t in range(t0, t0 + n)] for s in range(lo, hi)], dtype=torch.float64)


def _sharded_worker(rank, world, port, S, T, chunk, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ev, dropped = D.run_sharded(_source, S, T, chunk, batch_factory=_StandInBatch, R=16)
        if rank == 0:
            q.put((ev.tolist(), dropped))
        else:
            assert ev is None
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,S", [(2, 13), (4, 29), (8, 37), (8, 5)])
def test_run_sharded_gloo(world, S):
    T, chunk = 23, 10
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_worker, args=(r, world, port, S, T, chunk, q)) for r in range(world)]
    for p in procs:
        p.start()
    got, dropped = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    one = _StandInBatch(S)
    for t0 in range(0, T, chunk):
        one.update_chunk(_source(0, S, t0, min(chunk, T - t0)))
    want, _ = one.changepoints()
    assert got == want.tolist() and not dropped
    assert len(got) > 0
