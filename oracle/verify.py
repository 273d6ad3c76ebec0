"""Oracle for change-point verification and fail-slow pairing — TEST
INFRASTRUCTURE ONLY (same import rule as ``oracle/__init__.py``).

Plain numpy / Python loops, one event at a time, written from:
  * PAPER.md §4.2 "2) Change-point verification": "compares the average
    iteration time before and after each identified change-point, treating it as a
    jitter if the performance difference is less than 10%";
  * SPEC.md verify_changepoint: jitter iff |mean_after - mean_before| /
    mean_before < 0.10, otherwise a verified change point whose direction is the sign;
    window = min(20, samples available on each side);
  * SPEC.md detect_failslow: verified degrade/recover change points are
    paired into events; an unclosed degrade yields an open event; severity =
    mean_after / mean_before.
Readings where both are silent (V1-V5):
  V1 the boundary of a raw BOCD event (t, cp_index) is b = cp_index (first index of the
     MAP segment): before = x[b-w_b .. b-1], after = x[b .. b+w_a-1], w_b = min(W, b - t_lo),
     w_a = min(W, t_hi - b) over the x range [t_lo, t_hi) the caller provides;
  V2 a side with no sample -> status INSUFFICIENT (neither jitter nor verified);
  V3 direction: after > before -> DEGRADE (iteration time grew), after < before -> RECOVER;
  V4 pairing per series in time order: DEGRADE while idle opens an event (onset b,
     baseline = its mean_before, severity = mean_after/mean_before); DEGRADE while open
     keeps it open with severity = max(severity, mean_after/baseline) (ladder-shaped
     slowdowns); RECOVER while open closes it (recovery b); RECOVER while idle is
     ignored;
  V5 means are plain fp64 sums in index order divided by the count.
"""
from __future__ import annotations

import numpy as np

JITTER, DEGRADE, RECOVER, INSUFFICIENT = 0, 1, 2, 3


def verify(x, t_lo, events, window=20, rel=0.10, series_base=0):
    """x: [S][T] covering global steps [t_lo, t_lo + T).  events: iterable of
    (series, t, cp_index) with global series ids.  Returns a list of
    (series, t, cp_index, status, mean_before, mean_after, n_before, n_after)."""
    x = np.asarray(x, dtype=np.float64)
    T = x.shape[1]
    t_hi = t_lo + T
    out = []
    for (s, t, c) in events:
        row = x[int(s) - series_base]
        b = int(c)
        wb = max(0, min(window, b - t_lo))
        wa = max(0, min(window, t_hi - b))
        if wb == 0 or wa == 0:
            out.append((int(s), int(t), b, INSUFFICIENT, 0.0, 0.0, wb, wa))
            continue
        sb = 0.0
        for k in range(b - wb, b):            # V5: index order
            sb += float(row[k - t_lo])
        sa = 0.0
        for k in range(b, b + wa):
            sa += float(row[k - t_lo])
        mb, ma = sb / wb, sa / wa
        if abs(ma - mb) / mb < rel:             # P:778-779 "less than 10%"
            st = JITTER
        else:
            st = DEGRADE if ma > mb else RECOVER
        out.append((int(s), int(t), b, st, mb, ma, wb, wa))
    return out


def pair(verified):
    """verified: the output of verify(), in (series, t) order.  Returns fail-slow events
    (series, onset, recovery or -1, severity) in (series, onset) order (V4)."""
    out = []
    cur = None  # [series, onset, baseline, severity]
    last_s = None
    for (s, _t, b, st, mb, ma, _wb, _wa) in verified:
        if s != last_s:
            if cur is not None:
                out.append((cur[0], cur[1], -1, cur[3]))
            cur = None
            last_s = s
        if st == DEGRADE:
            if cur is None:
                cur = [s, b, mb, ma / mb]
            else:
                cur[3] = max(cur[3], ma / cur[2])
        elif st == RECOVER and cur is not None:
            out.append((cur[0], cur[1], b, cur[3]))
            cur = None
    if cur is not None:
        out.append((cur[0], cur[1], -1, cur[3]))
    return out
