"""N1 on the GPU: change-point verification and fail-slow pairing (falcon_verify_changepoints,
falcon_pair_failslow) against the oracle (oracle/verify.py) on the same raw events.

Verification sums in index order like the oracle, so status, window sizes and both means
must be bit-identical; pairing must return exactly the oracle's events.
"""
import numpy as np
import pytest

from oracle import verify as V
from paper_2410_12588_b200 import tracegen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2410_12588_b200 import bocd  # noqa: E402


def _raw_events(x, R, H, prior_cov, mask=3):
    S = x.shape[0]
    b = bocd.BocdBatch(S, R=R, hazard=H, prior_first_obs=True, prior_cov=prior_cov, event_mask=mask,
                       event_capacity=4096)
    b.update_chunk(torch.from_numpy(np.ascontiguousarray(x)).cuda())
    ev, dropped = b.changepoints()
    b.close()
    assert not dropped
    return ev


def _check_same(x, ev, t_lo=0, series_base=0, window=20):
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    got = bocd.verify_changepoints(xd, ev, t_lo=t_lo, series_base=series_base, window=window)
    want = V.verify(x, t_lo, [(int(e["series"]), int(e["t"]), int(e["cp_index"])) for e in ev],
                    window=window, series_base=series_base)
    assert len(got) == len(want)
    for g, w in zip(got, want):
        assert (int(g["series"]), int(g["t"]), int(g["cp_index"]), int(g["status"])) == w[:4]
        assert (int(g["n_before"]), int(g["n_after"])) == (w[6], w[7])
        if w[3] != V.INSUFFICIENT:
            assert g["mean_before"] == w[4] and g["mean_after"] == w[5]  # bit-identical (V5)
    pairs = bocd.pair_failslow(got)
    want_p = V.pair(want)
    assert [(int(p["series"]), int(p["onset"]), int(p["recovery"])) for p in pairs] == \
        [(s, o, r) for (s, o, r, _v) in want_p]
    assert np.array_equal(pairs["severity"], np.array([v for (_s, _o, _r, v) in want_p], dtype=np.float64))
    return got, pairs


@pytest.mark.parametrize("cfgname,S,T", [("C2", 64, 3000), ("C3", 256, 4000)])
def test_verify_and_pair_match_oracle(cfgname, S, T):
    cfg = tracegen.CONFIGS[cfgname]
    x = tracegen.generate(tracegen.make_spec(cfg), 0, S, 0, T)
    ev = _raw_events(x, cfg.R, cfg.hazard, cfg.prior_cov)
    assert len(ev) > 0
    got, pairs = _check_same(x, ev)
    st = got["status"]
    # the C-recipe episodes (>= 15% / >= 39% slowdowns) survive; raw jitter events are removed
    assert np.any(st == V.DEGRADE) and np.any(st == V.JITTER)
    assert len(pairs) > 0


def test_verify_window_edges_offsets_and_bad_series():
    rng = np.random.default_rng(11)
    x = rng.lognormal(0.0, 0.2, size=(6, 300))
    sb, t_lo = 100, 5000
    ev = np.zeros(7, dtype=bocd.EVENT_DTYPE)
    rows = [(100, 5100, 5050), (101, 5010, 5000), (101, 5299, 5299), (105, 5299, 5300),
            (103, 5200, 5190), (99, 5100, 5100), (106, 5100, 5100)]  # the last two: outside the shard
    for k, (s, t, c) in enumerate(rows):
        ev[k]["series"], ev[k]["t"], ev[k]["cp_index"], ev[k]["flags"] = s, t, c, 1
    xd = torch.from_numpy(x).cuda()
    got = bocd.verify_changepoints(xd, ev, t_lo=t_lo, series_base=sb, window=20)
    want = V.verify(x, t_lo, rows[:5], window=20, series_base=sb)
    for g, w in zip(got[:5], want):
        assert (int(g["status"]), int(g["n_before"]), int(g["n_after"])) == (w[3], w[6], w[7])
        if w[3] != V.INSUFFICIENT:
            assert g["mean_before"] == w[4] and g["mean_after"] == w[5]
    assert list(got["status"][5:]) == [V.INSUFFICIENT] * 2 and not got["n_before"][5:].any()


def test_pair_rejects_unsorted_input():
    v = np.zeros(3, dtype=bocd.VERIFIED_DTYPE)
    v["series"] = [0, 2, 1]
    v["status"] = V.DEGRADE
    v["mean_before"], v["mean_after"] = 1.0, 1.5
    with pytest.raises(bocd.N.FalconError):
        bocd.pair_failslow(v)
    assert len(bocd.pair_failslow(v[:0])) == 0
    assert len(bocd.verify_changepoints(torch.zeros((1, 4), dtype=torch.float64, device="cuda"),
                                        np.zeros(0, dtype=bocd.EVENT_DTYPE))) == 0


def test_spec_failslow_example_on_gpu():
    """one 30% slowdown over iterations 50-80 -> one event, onset in [50, 55],
    recovery in [80, 85], severity ~1.3 (GPU BOCD -> GPU verification -> GPU pairing)."""
    rng = np.random.default_rng(2410_12588)
    x = (1.0 + 0.01 * rng.standard_normal(200))[None, :]
    x[0, 50:81] *= 1.3
    ev = _raw_events(x, 256, 1 / 250, 0.05, mask=1)
    _got, pairs = _check_same(x, ev)
    assert len(pairs) == 1
    p = pairs[0]
    assert 50 <= p["onset"] <= 55 and 80 <= p["recovery"] <= 85 and p["severity"] == pytest.approx(1.3, rel=0.02)
