"""Oracle for ACF period detection and iteration-time derivation — TEST
INFRASTRUCTURE ONLY (same import rule as ``oracle/__init__.py``).

PAPER.md §4.2 "Iteration time analysis", written out directly:
  ACF(X)_k = sum_{t=1}^{L-k} (X_t - mu)(X_{t+k} - mu) / sum_{t=1}^{L} (X_t - mu)^2,
  mu = the mean of X (the L codes), k = 1 .. k_max;
  Period = argmin_k (ACF(X)_k >= M), M = 0.95;
  "the iteration time derives by calculating the time difference between a communication
  operation and its occurrence in the previous period": with SPEC S:120-122's
  anchors (the first call of each period block), duration_i = ts[(i+1) P] - ts[i P].
Readings (A1-A3): A1 the window is the whole sequence given (L = len(X));
A2 zero variance -> ACF 0 for every k, reported as a flag: period -1; A3 no
k <= k_max reaching M -> no period (0).  SPEC's pre-condition |codes| >= 2 k_max
raises ValueError (the insufficient-data error).  Plain numpy in fp64, one lag at a time.
"""
from __future__ import annotations

import numpy as np


def acf(codes, k_max):
    """ACF_k for k = 1..k_max of one code sequence (fp64).  Returns (acf[k_max], zero_var)."""
    x = np.asarray(codes, dtype=np.float64)
    L = len(x)
    mu = x.sum() / L
    y = x - mu
    den = float(np.sum(y * y))
    out = np.zeros(k_max)
    if den == 0.0:
        return out, True
    for k in range(1, k_max + 1):
        out[k - 1] = float(np.sum(y[: L - k] * y[k:])) / den
    return out, False


def detect_period(codes, k_max, M=0.95):
    """The smallest k in [1, k_max] with ACF_k >= M, 0 if none (A3), -1 for a zero-variance
    window (A2's flag).  Raises ValueError when len(codes) < 2 k_max."""
    if len(codes) < 2 * k_max:
        raise ValueError("insufficient data: detect_period needs |codes| >= 2 k_max")
    a, zero_var = acf(codes, k_max)
    if zero_var:
        return -1
    hit = np.nonzero(a >= M)[0]
    return int(hit[0]) + 1 if len(hit) else 0


def iteration_times(ts, period):
    """duration_i = ts[(i+1) P] - ts[i P] for every complete period block."""
    ts = np.asarray(ts, dtype=np.float64)
    if period <= 0:  # no period (0) or a zero-variance window (-1)
        return np.zeros(0)
    n = (len(ts) - 1) // period
    return np.array([ts[(i + 1) * period] - ts[i * period] for i in range(n)])
