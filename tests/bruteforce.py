"""Brute-force BOCD by enumeration of segmentations (test-only pin, mpmath).

This is the plain definition the recursion of PAPER.md Appendix A
 reaches exactly: a product-partition model in which a change
point follows each observation independently with probability H (the constant
change-point prior Pr(r_t | r_{t-1}), reading Q2), segments are i.i.d.
Gaussian with unknown mean/variance under a NIG prior (reading Q1), and the
run-length posterior after x_t is obtained by summing the joint weight of
every boundary pattern.  It shares nothing with ``oracle/``: segment
likelihoods use the closed-form NIG marginal likelihood, not the sequential
Student-t predictive.

Slot convention (reading Q7): slot r >= 1 = open segment of r observations
ending at x_t; slot 0 = a change point right after x_t.

Truncation (reading Q6):
  * DROP  — run lengths beyond R-1 are discarded: a segment that is still open
            has length <= R-1, a segment closed by a change point has length <= R.
  * MERGE — slot R-1 is the ">= R-1" bucket; inside a segment the k-th
            observation is predicted from the previous min(k-1, R-1)
            observations of that segment (windowed chain).
  * R >= t+2 makes both coincide with the untruncated model.
"""
from __future__ import annotations

import itertools

import mpmath


def log_ml(xs, mu0, k0, a0, b0):
    """Closed-form log marginal likelihood of xs under NIG(mu0, k0, a0, b0)."""
    n = len(xs)
    if n == 0:
        return mpmath.mpf(0)
    xb = sum(xs) / n
    kn = k0 + n
    an = a0 + mpmath.mpf(n) / 2
    bn = b0 + sum((v - xb) ** 2 for v in xs) / 2 + k0 * n * (xb - mu0) ** 2 / (2 * kn)
    return (mpmath.loggamma(an) - mpmath.loggamma(a0) + a0 * mpmath.log(b0) - an * mpmath.log(bn)
            + mpmath.log(k0 / kn) / 2 - n * mpmath.log(2 * mpmath.pi) / 2)


def posterior(x, R, H, mu0, k0, a0, b0, mode, dps=40, decisions=False):
    """Return (logR[t][r] as floats, cumulative log evidence per t) for t = 0..len(x)-1.

    decisions=True also returns, per t, the decision quantities of reading Q4/Q5
    ("likelihood of r_t = 0 ... exceeds 0.9"; P:762-770 MAP run length),
    each defined directly on the segmentations rather than from the slot values:
      * p_new_t = Pr(x_t opens a new segment | x_{0..t}, the open segment fits the
        truncation) = W(last segment has length 1) / W(every admissible pattern whose
        open segment is a growth slot: length <= R-1 under DROP, any under MERGE), W the
        summed pattern weights without the change-point factor that follows x_t.  (Slot 1
        of MERGE with R = 2 is the ">= 1" bucket: then "length 1" means "in slot 1".)
      * map_t = the growth slot r >= 1 of largest posterior mass (ties -> smaller r) and
        margin_t = its log mass minus the next largest log mass over r >= 1, r != map_t.
    """
    mpmath.mp.dps = dps
    xs = [mpmath.mpf(float(v)) for v in x]
    mu0, k0, a0, b0 = (mpmath.mpf(float(v)) for v in (mu0, k0, a0, b0))
    H = mpmath.mpf(float(H))
    lH, l1H = mpmath.log(H), mpmath.log(1 - H)
    n = len(xs)
    W = R - 1
    cache = {}

    def seg(a, b):  # log likelihood of segment x[a..b] (inclusive)
        key = (a, b)
        if key not in cache:
            if mode == "merge":
                tot = mpmath.mpf(0)
                for k in range(a, b + 1):
                    lo = max(a, k - W)
                    tot += log_ml(xs[lo:k + 1], mu0, k0, a0, b0) - log_ml(xs[lo:k], mu0, k0, a0, b0)
                cache[key] = tot
            else:
                cache[key] = log_ml(xs[a:b + 1], mu0, k0, a0, b0)
        return cache[key]

    out, evid, dec = [], [], []
    for t in range(n):
        acc = [[] for _ in range(R)]
        w_new, w_open = [], []
        for bits in itertools.product((0, 1), repeat=t):
            starts = [0] + [k + 1 for k in range(t) if bits[k]]
            ends = starts[1:] + [t + 1]
            lens = [e - s for s, e in zip(starts, ends)]
            lw = sum(lH if b else l1H for b in bits)
            lw += sum(seg(s, e - 1) for s, e in zip(starts, ends))
            last = lens[-1]
            if mode == "drop":
                if any(L > R for L in lens[:-1]):
                    continue
                if last <= R:
                    acc[0].append(lH + lw)
                if last <= R - 1:
                    acc[last].append(l1H + lw)
                    w_open.append(lw)
                    if last == 1:
                        w_new.append(lw)
            else:
                acc[0].append(lH + lw)
                acc[min(last, R - 1)].append(l1H + lw)
                w_open.append(lw)
                if min(last, R - 1) == 1:
                    w_new.append(lw)
        slot = [mpmath.log(mpmath.fsum(mpmath.exp(v) for v in a)) if a else None for a in acc]
        live = [v for v in slot if v is not None]
        tot = mpmath.log(mpmath.fsum(mpmath.exp(v) for v in live))
        out.append([float(v - tot) if v is not None else float("-inf") for v in slot])
        evid.append(float(tot))
        if decisions:
            lse = lambda a: mpmath.log(mpmath.fsum(mpmath.exp(v) for v in a))
            p_new = mpmath.exp(lse(w_new) - lse(w_open)) if w_new else mpmath.mpf(0)
            grow = [(slot[r], r) for r in range(1, R) if slot[r] is not None]
            best = max(grow, key=lambda vr: (vr[0], -vr[1]))
            rest = [v for v, r in grow if r != best[1]]
            margin = best[0] - max(rest) if rest else mpmath.inf
            dec.append({"p_new": float(p_new), "map": best[1], "margin": float(margin)})
    return (out, evid, dec) if decisions else (out, evid)
