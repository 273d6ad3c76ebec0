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


def evaluate(spec, cfg, T: int, min_len: int = 20, event_capacity: int = 8192, device="cuda"):
    """Scores of raw BOCD and BOCD+V on one labelled synthetic suite (tracegen spec over its
    S series x T steps), every detector running on the GPU through the C ABI: the BOCD batch
    (PROB events, p_new > 0.9 of P:770, and MAP resets), falcon_verify_changepoints (the 10%
    rule of P:772-779) and falcon_pair_failslow.  Returns the dict tools/detection_accuracy.py
    prints (Tables 5-6 scores per detector)."""
    import torch

    from . import _native as N, bocd
    S = spec.n_series
    x = torch.empty((S, T), dtype=torch.float64, device=device)
    bocd.DeviceTrace(spec, device).generate(x, 0, 0)
    b = bocd.BocdBatch(S, R=cfg.R, hazard=cfg.hazard, prior_first_obs=True, prior_cov=cfg.prior_cov,
                       event_mask=3, event_capacity=event_capacity)
    b.update_chunk(x)
    ev, dropped = b.changepoints()
    b.close()
    truth, onset = series_truth(spec, 0, T, min_len=min_len)
    out = {"config": cfg.name, "sigma": float(spec.sigma[0]), "series": S, "steps": T, "R": cfg.R,
           "slowed_series": int(truth.sum()), "events_dropped": bool(dropped)}
    for label, mask in (("prob", 1), ("prob_mapreset", 3)):
        raw = ev[(ev["flags"] & mask) != 0]
        first_raw = first_flag(raw["series"], raw["t"], S)
        ver = bocd.verify_changepoints(x, raw, t_lo=0)
        pairs = bocd.pair_failslow(ver)
        # a verified change point is known once its 20-sample after-window is complete
        deg = ver[ver["status"] == N.CP_DEGRADE]
        t_known = np.maximum(deg["t"], deg["cp_index"] + 19)
        first_v = first_flag(deg["series"], t_known, S)
        flagged_v = np.zeros(S, dtype=bool)
        flagged_v[pairs["series"]] = True  # every fail-slow event starts at a verified DEGRADE
        out["bocd_" + label] = {**confusion(first_raw >= 0, truth), "raw_events": int(len(raw)),
                                "delay_steps": latency(first_raw, onset, truth)}
        out["bocd_v_" + label] = {**confusion(flagged_v, truth), "failslow_events": int(len(pairs)),
                                  "delay_steps": latency(np.where(flagged_v, first_v, -1), onset, truth)}
    return out
