"""Pins of the suspicious-group oracle (oracle/groups.py): the SPEC examples
(S:207-210), numpy's median, permutation and scale invariance."""
import numpy as np
import pytest

from oracle import groups as G


@pytest.mark.parametrize("row,med,flags", [
    ([10, 10, 10, 12], 10.0, [False, False, False, True]),    # S:208 (median 10, cutoff 11)
    ([7, 7, 7, 7], 7.0, [False] * 4),                         # S:209 all equal -> empty
    ([10, 10, 11, 11], 10.5, [False] * 4),                    # S:210 (median 10.5, cutoff 11.55)
    ([5.0], 5.0, [False]),
    ([1.0, 3.0], 2.0, [False, True]),                         # 3 > 2.2
    ([1.0, 2.0, 2.2, 2.21], 2.1, [False, False, False, False]),  # 2.21 < 1.1 * 2.1 = 2.31
])
def test_spec_examples(row, med, flags):
    (m, f), = G.classify([row])
    assert m == pytest.approx(med, rel=1e-15) and f == flags


def test_median_matches_numpy_and_invariances():
    rng = np.random.default_rng(9)
    for n in (1, 2, 3, 8, 31, 256, 1001):
        row = rng.lognormal(0.0, 0.3, size=n)
        (m, f), = G.classify([row])
        assert m == np.median(row)
        perm = rng.permutation(n)
        (m2, f2), = G.classify([row[perm]])
        assert m2 == m and [f[k] for k in perm] == f2
        for c in (0.5, 4.0):  # powers of two: exact scaling, identical decisions
            (m3, f3), = G.classify([row * c])
            assert m3 == m * c and f3 == f
