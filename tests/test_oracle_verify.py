"""Pins of the verification / pairing oracle (oracle/verify.py).

The paper fixes only the rule (jitter iff the before/after mean difference is
below 10%); SPEC S:136-153 gives worked examples; the means are checked against numpy's
mean over explicit slices, and the end-to-end examples run the BOCD oracle.
"""
import numpy as np
import pytest

from oracle import verify as V


def _one(before, after, n=20, window=20):
    x = np.array([[before] * n + [after] * n], dtype=np.float64)
    return V.verify(x, 0, [(0, n, n)], window=window)[0]


@pytest.mark.parametrize("before,after,status", [
    (1.00, 1.05, V.JITTER),    # S:141 "before=1.00, after=1.05 -> jitter"
    (1.00, 1.20, V.DEGRADE),   # S:142 "before=1.00, after=1.20 -> degrade"
    (1.00, 1.00, V.JITTER),    # S:143 "before==after -> jitter"
    (1.20, 1.00, V.RECOVER),   # direction by sign
    (10.0, 11.0, V.DEGRADE),   # exactly 10%: "less than 10%" is strict
    (10.0, 10.99, V.JITTER),
])
def test_spec_examples(before, after, status):
    r = _one(before, after)
    assert r[3] == status
    assert r[4] == pytest.approx(before, rel=1e-15) and r[5] == pytest.approx(after, rel=1e-15)


def test_means_match_numpy_slices_and_window_truncation():
    rng = np.random.default_rng(3)
    x = rng.lognormal(0.0, 0.2, size=(3, 200))
    t_lo = 1000
    ev = [(0, 1100, 1050), (1, 1010, 1005), (2, 1199, 1190), (2, 1199, 1000), (1, 1150, 1200)]
    out = V.verify(x, t_lo, ev, window=20)
    for (s, t, c), (s2, t2, b, st, mb, ma, wb, wa) in zip(ev, out):
        assert (s2, t2, b) == (s, t, c)
        k = c - t_lo
        assert wb == min(20, k) and wa == min(20, 200 - k)
        if wb == 0 or wa == 0:
            assert st == V.INSUFFICIENT
            continue
        assert mb == pytest.approx(np.mean(x[s, k - wb:k]), rel=1e-14)
        assert ma == pytest.approx(np.mean(x[s, k:k + wa]), rel=1e-14)
        want = V.JITTER if abs(ma - mb) / mb < 0.1 else (V.DEGRADE if ma > mb else V.RECOVER)
        assert st == want


def test_scale_invariance():
    """multiplying all durations by c > 0 preserves the classification."""
    rng = np.random.default_rng(5)
    x = rng.lognormal(0.0, 0.15, size=(4, 120))
    ev = [(s, 60, c) for s in range(4) for c in (20, 40, 60, 80, 100)]
    base = [r[3] for r in V.verify(x, 0, ev)]
    for c in (0.25, 8.0, 3.0e-3):  # powers of two are exact; 3e-3 checks the generic case
        got = [r[3] for r in V.verify(x * c, 0, ev)]
        assert got == base


def test_pairing_state_machine():
    D, Rc, J = V.DEGRADE, V.RECOVER, V.JITTER
    rows = [  # (series, t, b, status, mean_before, mean_after, nb, na)
        (0, 10, 10, D, 1.0, 1.3, 20, 20), (0, 30, 30, J, 1.3, 1.31, 20, 20), (0, 50, 50, Rc, 1.3, 1.0, 20, 20),
        (0, 70, 70, Rc, 1.0, 0.8, 20, 20),                                     # recover while idle: ignored
        (0, 90, 90, D, 1.0, 1.2, 20, 20), (0, 95, 95, D, 1.2, 1.5, 20, 20),    # ladder: severity 1.5/1.0
        (1, 5, 5, D, 2.0, 3.0, 5, 20),                                         # open at the end of series 1
        (2, 7, 7, Rc, 2.0, 1.0, 7, 20),
    ]
    got = V.pair(rows)
    assert got == [(0, 10, 50, 1.3), (0, 90, -1, 1.5), (1, 5, -1, 1.5)]


def _bocd_failslow(oracle_mod, x, window=20, mask=1):
    res = oracle_mod.run(x, 256, 1 / 250, prior_first_obs=True, prior_cov=0.05)
    raw = [(s, t, c) for (s, t, c, f, p) in res.events(mask)]
    return V.pair(V.verify(x, 0, raw, window=window)), raw


def test_spec_failslow_examples(oracle_mod):
    """S:150-152 end to end (BOCD oracle -> verification -> pairing)."""
    rng = np.random.default_rng(2410_12588)
    T = 200
    base = 1.0 + 0.01 * rng.standard_normal(T)
    clean = base[None, :]
    ev, _ = _bocd_failslow(oracle_mod, clean)
    assert ev == []                                                   # "clean series -> empty list"
    one = base.copy()
    one[50:81] *= 1.3
    ev, raw = _bocd_failslow(oracle_mod, one[None, :])
    assert len(ev) == 1, (ev, raw)                                    # "one 30% slowdown iters 50-80"
    s, onset, rec, sev = ev[0]
    assert 50 <= onset <= 55 and 80 <= rec <= 85 and sev == pytest.approx(1.3, rel=0.02)
    two = base.copy()
    two[40:70] *= 1.3
    two[120:150] *= 1.5
    ev, raw = _bocd_failslow(oracle_mod, two[None, :])
    assert [(o, r) for (_s, o, r, _v) in ev] == sorted((o, r) for (_s, o, r, _v) in ev)  # in order
    assert len(ev) == 2 and 40 <= ev[0][1] <= 45 and 120 <= ev[1][1] <= 125, (ev, raw)


def test_verification_removes_jitter_false_positives(oracle_mod):
    """raw BOCD flags jitters; verification drops those below 10%.  Raw change
    points = PROB | MAPRESET events (the MAP resets also flag the 5% bump)."""
    rng = np.random.default_rng(7)
    T = 400
    x = 1.0 + 0.01 * rng.standard_normal(T)
    x[100:130] *= 1.05   # a 5% bump: raw change points, never a fail-slow
    x[250:300] *= 1.25   # a real 25% slowdown
    ev, raw = _bocd_failslow(oracle_mod, x[None, :], mask=3)
    assert any(100 <= c <= 133 for (_s, _t, c) in raw)  # the bump is a raw change point ...
    assert ev == [(0, 250, 300, pytest.approx(1.25, rel=0.02))], (ev, raw)  # ... but not an event
