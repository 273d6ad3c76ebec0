"""Oracle for suspicious-group classification — TEST INFRASTRUCTURE ONLY
(same import rule as ``oracle/__init__.py``).

PAPER.md §4.3 "Profiling": per-group data-transfer times are measured with CUDA
events and "communication groups with data transfer time longer than 1.1x median value are
classified as suspicious".  SPEC.md classify_groups: suspicious iff
transfer_time > 1.1 x median(transfer_time), median of an even count = mean of the two
middle values.  Plain Python: sort, pick, compare (one batch = one profiling round).
"""
from __future__ import annotations


def median(values):
    v = sorted(float(a) for a in values)
    n = len(v)
    if n % 2 == 1:
        return v[n // 2]
    return (v[n // 2 - 1] + v[n // 2]) / 2.0


def classify(batches, factor=1.1):
    """batches: iterable of per-group transfer-time lists.  Returns, per batch,
    (median, [suspicious flags]) with flag = t > factor * median (strict, "longer")."""
    out = []
    for row in batches:
        m = median(row)
        cut = factor * m
        out.append((m, [float(t) > cut for t in row]))
    return out
