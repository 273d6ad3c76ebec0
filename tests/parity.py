"""Parity comparators (readings Q9, Q10, Q12) — test-only helpers.

Tolerances (BASELINE.json north_star): log posteriors within 1e-9 absolute of
the fp64 oracle; change-point indices bit-exact except where the oracle's MAP
margin is below 1e-6 (or, for the PROB flag, |p_new - theta| < 1e-6).
"""
from __future__ import annotations

import numpy as np

TOL_LOG = 1e-9      # |Delta log R|, |Delta log Z|
LIVE = -50.0        # slots with oracle log R >= -50 are compared at TOL_LOG (Q12)
DEAD_CEIL = -40.0   # slots below -50 in the oracle must stay below -40 on the GPU
MARGIN = 1e-6       # MAP exemption (Q9)
PMARGIN = 1e-6      # threshold exemption (Q10)


def compare_logR(gpu, ref, tol=TOL_LOG):
    """Returns max |Delta| over live slots; asserts the dead-slot rule."""
    gpu = np.asarray(gpu)
    ref = np.asarray(ref)
    live = ref >= LIVE
    assert np.all(np.isfinite(gpu[live])), "non-finite GPU value on a live slot"
    d = np.abs(gpu[live] - ref[live])
    worst = float(d.max()) if d.size else 0.0
    assert worst <= tol, f"max |dlogR| on live slots = {worst:.3e} > {tol:.1e}"
    dead = ~live
    if np.any(dead):
        bad = gpu[dead] >= DEAD_CEIL
        assert not np.any(bad), f"{int(bad.sum())} dead slots above {DEAD_CEIL} on the GPU"
    return worst


def exempt_steps(margin, p_new, theta):
    """Steps whose discrete outputs may legitimately differ: MAP near-ties at t or t-1
    (MAPRESET reads r*_{t-1}), or p_new within PMARGIN of theta."""
    m = np.asarray(margin) < MARGIN
    mprev = np.zeros_like(m)
    mprev[..., 1:] = m[..., :-1]
    return m | mprev | (np.abs(np.asarray(p_new) - theta) < PMARGIN)


def compare_steps(g_map, g_pnew, g_logz, res, theta, tol=TOL_LOG):
    """Per-step outputs vs an OracleResult.  Returns a dict of statistics."""
    ex = exempt_steps(res.margin, res.p_new, theta)
    mism = (np.asarray(g_map) != res.map_rl) & ~(np.asarray(res.margin) < MARGIN)
    assert not np.any(mism), f"MAP run length differs at {np.argwhere(mism)[:5].tolist()}"
    dz = np.abs(np.asarray(g_logz) - res.log_z)
    assert dz.max() <= tol, f"max |dlogZ| = {dz.max():.3e}"
    dp = np.abs(np.asarray(g_pnew) - res.p_new)
    assert dp.max() <= tol, f"max |dp_new| = {dp.max():.3e}"
    return {"max_dlogz": float(dz.max()), "max_dpnew": float(dp.max()),
            "exempt_steps": int(ex.sum())}


def compare_events(gpu_events, res, theta, mask):
    """GPU events (structured array) vs oracle flags, outside exempt steps."""
    ex = exempt_steps(res.margin, res.p_new, theta)
    # event records carry the requested flag bits only (include/falcon_bocd.h)
    want = {(s, t, c, f & mask) for (s, t, c, f, _p) in res.events(mask) if not ex[s, t]}
    got = {(int(e["series"]), int(e["t"]), int(e["cp_index"]), int(e["flags"]))
           for e in gpu_events if not ex[int(e["series"]), int(e["t"])]}
    assert got == want, f"events differ: missing {sorted(want - got)[:5]}, extra {sorted(got - want)[:5]}"
    return len(want)


STATS = {}


def record(name, stats):
    """Collect per-case parity statistics (dumped by conftest when PARITY_STATS is set)."""
    STATS[name] = stats
