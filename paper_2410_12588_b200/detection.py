"""Detection-accuracy bookkeeping for labelled synthetic traces (without the
paper's SlideWindow comparison system).

PAPER.md Tables 5-6 score detectors per job: a job is positive when it was
slowed, a detector is positive when it reports a fail-slow; accuracy, FPR = FP/(FP+TN) and
FNR = FN/(FN+TP).  Here the unit is one synthetic series (a rank or a link, tracegen
recipes) and the ground truth is the generator's injected episode table, so the scores
describe this library's detectors (raw BOCD change points; BOCD + the 10% verification of
P:772-779 and fail-slow pairing) on synthetic data.  They are not the paper's numbers:
its labelled traces were not released.  Host logic only (numpy); the detectors run
through the C ABI (tools/detection_accuracy.py).
"""
from __future__ import annotations

import numpy as np


def series_truth(spec, t_lo: int, t_hi: int, min_len: int = 1):
    """Per series: (slowed, first onset) for the injected episodes overlapping [t_lo, t_hi)
    by at least min_len steps.  Returns (bool[S], int64[S] with -1 where not slowed)."""
    S = spec.n_series
    slowed = np.zeros(S, dtype=bool)
    onset = np.full(S, -1, dtype=np.int64)
    for s in range(S):
        for a, b, _sev in spec.episodes(s):
            lo, hi = max(a, t_lo), min(b, t_hi)
            if hi - lo >= min_len:
                slowed[s] = True
                onset[s] = lo if onset[s] < 0 else min(onset[s], lo)
    return slowed, onset


def first_flag(series_ids, times, S: int):
    """First flagged step per series from event arrays (-1: never flagged)."""
    first = np.full(S, -1, dtype=np.int64)
    for s, t in zip(np.asarray(series_ids, dtype=np.int64), np.asarray(times, dtype=np.int64)):
        if first[s] < 0 or t < first[s]:
            first[s] = t
    return first


def confusion(flagged, truth):
    """Accuracy, FPR and FNR as in PAPER.md Tables 5-6."""
    flagged = np.asarray(flagged, dtype=bool)
    truth = np.asarray(truth, dtype=bool)
    tp = int(np.sum(flagged & truth))
    fp = int(np.sum(flagged & ~truth))
    tn = int(np.sum(~flagged & ~truth))
    fn = int(np.sum(~flagged & truth))
    n = tp + fp + tn + fn
    return {"tp": tp, "fp": fp, "tn": tn, "fn": fn,
            "accuracy": (tp + tn) / n if n else float("nan"),
            "fpr": fp / (fp + tn) if fp + tn else float("nan"),
            "fnr": fn / (fn + tp) if fn + tp else float("nan")}


def latency(first, onset, truth):
    """Steps from the first injected onset to the first flag, over true positives whose first
    flag is at or after the onset (a flag before the onset is a false alarm, not a detection)."""
    first = np.asarray(first, dtype=np.int64)
    onset = np.asarray(onset, dtype=np.int64)
    ok = np.asarray(truth, dtype=bool) & (first >= 0) & (first >= onset)
    d = (first - onset)[ok]
    if d.size == 0:
        return {"n": 0}
    return {"n": int(d.size), "median": float(np.median(d)), "p90": float(np.percentile(d, 90)),
            "max": int(d.max())}
