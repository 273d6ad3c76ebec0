"""Seeded synthetic iteration-time / link-time traces (input generator).

This module holds NONE of the method's arithmetic: it only produces the
observations x[s, t] that both the CUDA path and the CPU oracle consume.  It
is the single shared piece between the two sides.

Recipe (after SURVEY.md §8(d)):

    x[s, t] = b_s * exp(sigma_s * z[s, t] + gamma * eta[t] + sum_{episodes e of s active at t} log sev_e)

* z and eta are standard normals from a counter-based hash keyed by
  (seed, global series id, t) — splitmix64 + Box-Muller — so every shard and
  every chunk reproduces exactly the same values.  The device twin
  (``csrc/tracegen.cu``, ``falcon_trace_generate``) implements the same
  counter generator; it agrees with this numpy twin to a few ulp
  (transcendental rounding), and the parity tests always feed both sides the
  same bytes.
* Episodes (fail-slow injections, "manually injected fail-slows") are
  drawn once per config from a seeded numpy generator over the GLOBAL series
  set, so shards slice the same table.

The five workloads follow BASELINE.json ``configs`` and the paper's workload
shapes.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_GOLD = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)
ETA_SERIES = 0xFFFFFFFFFFFFFFFF  # series key used for the common term eta[t]


def splitmix64(z):
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + _GOLD
        z = (z ^ (z >> np.uint64(30))) * _C1
        z = (z ^ (z >> np.uint64(27))) * _C2
    return z ^ (z >> np.uint64(31))


def uniform01(seed: int, series, t, stream: int):
    """u in (0, 1): ((h >> 11) + 0.5) * 2^-53 with h = hash(seed, series, 2t + stream)."""
    k0 = splitmix64(np.uint64(seed))
    k1 = splitmix64(k0 ^ np.asarray(series, dtype=np.uint64))
    with np.errstate(over="ignore"):
        c = np.asarray(t, dtype=np.uint64) * np.uint64(2) + np.uint64(stream)
    h = splitmix64(k1 ^ c)
    return ((h >> np.uint64(11)).astype(np.float64) + 0.5) * (2.0 ** -53)


def std_normal(seed: int, series, t):
    """Box-Muller on two counter-based uniforms."""
    u1 = uniform01(seed, series, t, 0)
    u2 = uniform01(seed, series, t, 1)
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)


@dataclass
class TraceSpec:
    """Per-series parameters + CSR episode table for the global series set."""
    seed: int
    n_series: int
    T: int
    b: np.ndarray          # [S] baseline iteration / transfer time (s)
    sigma: np.ndarray      # [S] log-normal noise scale
    gamma: float           # scale of the common (cluster-wide) term eta[t]
    ep_off: np.ndarray     # [S+1] int64 CSR offsets
    ep_start: np.ndarray   # [E] int64, first affected step
    ep_end: np.ndarray     # [E] int64, one past the last affected step
    ep_logsev: np.ndarray  # [E] log of the slowdown factor

    def episodes(self, s: int):
        a, b = int(self.ep_off[s]), int(self.ep_off[s + 1])
        return list(zip(self.ep_start[a:b].tolist(), self.ep_end[a:b].tolist(),
                        np.exp(self.ep_logsev[a:b]).tolist()))


def generate(spec: TraceSpec, s0: int = 0, count: int | None = None, t0: int = 0,
             T: int | None = None) -> np.ndarray:
    """x[s0:s0+count, t0:t0+T] as a fresh fp64 array (numpy twin of falcon_trace_generate)."""
    count = spec.n_series - s0 if count is None else count
    T = spec.T - t0 if T is None else T
    sids = np.arange(s0, s0 + count, dtype=np.uint64)[:, None]
    ts = np.arange(t0, t0 + T, dtype=np.uint64)[None, :]
    z = std_normal(spec.seed, sids, ts)
    eta = std_normal(spec.seed, np.uint64(ETA_SERIES), ts) if spec.gamma != 0.0 else 0.0
    e = spec.sigma[s0:s0 + count, None] * z + spec.gamma * eta
    tt = np.arange(t0, t0 + T, dtype=np.int64)
    for i, s in enumerate(range(s0, s0 + count)):
        for k in range(int(spec.ep_off[s]), int(spec.ep_off[s + 1])):
            m = (tt >= spec.ep_start[k]) & (tt < spec.ep_end[k])
            e[i, m] += spec.ep_logsev[k]
    return spec.b[s0:s0 + count, None] * np.exp(e)


@dataclass
class BocdConfig:
    """One BASELINE.json workload: trace recipe + BOCD hyper-parameters (readings Q2, Q3)."""
    name: str
    n_series: int
    T: int
    R: int
    hazard: float = 1.0 / 250.0
    kappa0: float = 1.0
    alpha0: float = 1.0
    prior_cov: float = 0.05          # beta0 = alpha0 * (prior_cov * x_0)^2, mu0 = x_0
    threshold: float = 0.9
    seed: int = 241012588
    extra: dict = field(default_factory=dict)


def _csr(lists, S):
    off = np.zeros(S + 1, np.int64)
    st, en, ls = [], [], []
    for s in range(S):
        eps = lists.get(s, [])
        off[s + 1] = off[s] + len(eps)
        for a, b, sev in eps:
            st.append(a); en.append(b); ls.append(np.log(sev))
    return off, np.array(st, np.int64), np.array(en, np.int64), np.array(ls, np.float64)


def _csr_vectorised(owner, start, end, logsev, S):
    order = np.lexsort((start, owner))
    owner, start, end, logsev = owner[order], start[order], end[order], logsev[order]
    off = np.zeros(S + 1, np.int64)
    np.add.at(off, owner + 1, 1)
    return np.cumsum(off), start.astype(np.int64), end.astype(np.int64), logsev


def make_spec(cfg: BocdConfig, n_series: int | None = None, T: int | None = None,
              sigma: float | None = None) -> TraceSpec:
    """Build the trace spec for a workload (optionally overriding S, T or sigma)."""
    S = cfg.n_series if n_series is None else n_series
    T = cfg.T if T is None else T
    seed = cfg.seed + {"C1": 1, "C2": 2, "C3": 3, "C4": 4, "C5": 5}.get(cfg.name, 0)
    rng = np.random.Generator(np.random.Philox(seed))
    kind = cfg.extra.get("kind", cfg.name)
    if kind == "C1":
        # 1 series x 1,000 iterations, one injected 1.5x step slowdown at t=600 (BJ configs[0]).
        sg = 0.02 if sigma is None else sigma
        lists = {s: [(600, T, 1.5)] for s in range(S)} if T > 600 else {}
        off, st, en, ls = _csr(lists, S)
        return TraceSpec(seed, S, T, np.full(S, 1.0), np.full(S, sg), 0.0, off, st, en, ls)
    if kind == "C2":
        # 1024-GPU hybrid-parallel job: 6 culprit ranks with one compute fail-slow each
        # (severity ~1.2x, P:405 / P:428; 30 s-60 min at 2 s/iter, P:35 / P:372).  Synchronous
        # training propagates a straggler to every rank.
        sg = 0.015 if sigma is None else sigma
        sev = rng.uniform(1.15, 1.25, 6)
        dur = np.exp(rng.uniform(np.log(15), np.log(1800), 6)).astype(np.int64)
        onset = (rng.random(6) * np.maximum(T - dur, 1)).astype(np.int64)
        eps = [(int(a), int(min(a + d, T)), float(v)) for a, d, v in zip(onset, dur, sev)]
        off, st, en, ls = _csr({s: eps for s in range(S)}, S)
        return TraceSpec(seed, S, T, np.full(S, 2.0), np.full(S, sg), 0.005, off, st, en, ls)
    # C3 / C4 / C5: per-link communication series on a large RoCE cluster.
    # b_s ~ U(0.05, 0.5) s; CoV 0.29 for RDMA -> sigma = 0.284;
    # 40% of links slowed, Poisson(1.5) episodes each, severity
    # log-uniform 1.39x-6.7x, duration log-uniform
    # 10 min-10 h at 1.75 s/iter = 343-20,571 steps.
    sg = 0.284 if sigma is None else sigma
    b = rng.uniform(0.05, 0.5, S)
    slowed = rng.random(S) < 0.4
    n_ep = np.where(slowed, np.maximum(1, rng.poisson(1.5, S)), 0)
    E = int(n_ep.sum())
    owner = np.repeat(np.arange(S, dtype=np.int64), n_ep)
    sev = np.exp(rng.uniform(np.log(1.39), np.log(6.7), E))
    dur = np.exp(rng.uniform(np.log(343), np.log(20571), E)).astype(np.int64)
    onset = (rng.random(E) * T).astype(np.int64)
    end = np.minimum(onset + dur, T)
    off, st, en, ls = _csr_vectorised(owner, onset, end, np.log(sev), S)
    return TraceSpec(seed, S, T, b, np.full(S, sg), 0.0, off, st, en, ls)


CONFIGS = {
    "C1": BocdConfig("C1", 1, 1000, 256, prior_cov=0.05),
    "C2": BocdConfig("C2", 1024, 10000, 512, prior_cov=0.05),
    "C3": BocdConfig("C3", 32768, 100000, 1024, prior_cov=0.3),
    "C4": BocdConfig("C4", 100000, 100000, 4096, prior_cov=0.3),
    "C5": BocdConfig("C5", 10240, 10000, 1024, prior_cov=0.3, extra={"kind": "C5"}),
}
