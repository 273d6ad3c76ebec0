"""Pins of the ACF / period oracle (oracle/acf.py): closed forms of the
paper's biased ACF on alternating and block-periodic codes, numpy's
correlate, the zero-variance case, and the SPEC detect_period / iteration_times examples."""
import numpy as np
import pytest

from oracle import acf as A


def test_alternating_closed_forms():
    """codes 1,2,1,2,... (L = 100): ACF_2 = (L-2)/L = 0.98, ACF_1 = -(L-1)/L."""
    x = np.tile([1, 2], 50)
    a, zv = A.acf(x, 4)
    assert not zv
    assert a[1] == pytest.approx(98 / 100, abs=1e-15)
    assert a[0] == pytest.approx(-99 / 100, abs=1e-15)
    assert a[3] == pytest.approx(96 / 100, abs=1e-15)   # (L-k)/L at every even lag


def test_matches_numpy_correlate():
    rng = np.random.default_rng(4)
    x = rng.integers(0, 9, size=777).astype(np.float64)
    a, _ = A.acf(x, 50)
    y = x - x.mean()
    full = np.correlate(y, y, mode="full")[len(x) - 1:] / np.dot(y, y)
    np.testing.assert_allclose(a, full[1:51], rtol=0, atol=1e-13)


def test_zero_variance_and_none():
    a, zv = A.acf(np.full(64, 3.0), 8)
    assert zv and not a.any() and A.detect_period(np.full(64, 3.0), 8) == -1  # S:104-105 flag
    with pytest.raises(ValueError):
        A.detect_period(np.arange(20), 11)  # |codes| < 2 k_max
    rng = np.random.default_rng(1)
    assert A.detect_period(rng.integers(0, 50, size=4096), 64) == 0      # S:114 random codes -> none


def test_spec_period_examples():
    blk = np.tile([11, 22, 33, 44], 32)                                   # S:112 [A,B,C,D]x32 -> 4
    assert A.detect_period(blk, 16) == 4
    # a 7-call block of collective-op codes (RS/AG/AR-like alphabet of 5), 1% of the
    # codes replaced by another op code -> period 7
    for seed in range(4):
        rng = np.random.default_rng(seed)
        b7 = np.tile([1, 2, 3, 2, 4, 1, 5], 300)
        flip = rng.random(len(b7)) < 0.01
        b7[flip] = rng.integers(1, 6, size=flip.sum())
        assert A.detect_period(b7, 32) == 7


def test_iteration_times_examples():
    ts = np.arange(0, 41, dtype=np.float64) * 0.25                       # 4-call period, 1 s per block
    assert np.array_equal(A.iteration_times(ts, 4), np.ones(10))
    ts2 = ts.copy()
    ts2[12:] += 0.5                                                      # one block stretched to 1.5 s
    d = A.iteration_times(ts2, 4)
    assert list(d).count(1.5) == 1 and np.sum(d != 1.0) == 1
