"""N2 on the GPU (falcon_detect_period, falcon_iteration_times) against the oracle
(oracle/acf.py), and the tracking chain of PAPER §4.2 end to end on the GPU: call codes ->
period -> iteration times -> BOCD -> verification -> fail-slow events."""
import numpy as np
import pytest

from oracle import acf as A

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2410_12588_b200 import bocd  # noqa: E402


def _traces(S, L, seed):
    """Per-rank call-signature codes: a random block of 3..12 collective-op codes repeated,
    1% of calls replaced by another op code; some ranks aperiodic."""
    rng = np.random.default_rng(seed)
    codes = np.empty((S, L), dtype=np.int32)
    for s in range(S):
        if s % 7 == 6:
            codes[s] = rng.integers(1, 9, size=L)
            continue
        P = int(rng.integers(3, 13))
        blk = rng.integers(1, 9, size=P)
        row = np.tile(blk, L // P + 1)[:L]
        flip = rng.random(L) < 0.01
        row[flip] = rng.integers(1, 9, size=flip.sum())
        codes[s] = row
    return codes


@pytest.mark.parametrize("S,L,kmax", [(37, 512, 32), (64, 4096, 256), (5, 8192, 1000)])
def test_acf_and_period_match_oracle(S, L, kmax):
    codes = _traces(S, L, S + L)
    period, acf = bocd.detect_period(torch.from_numpy(codes).cuda(), kmax, with_acf=True)
    period, acf = period.cpu().numpy(), acf.cpu().numpy()
    for s in range(S):
        a, _ = A.acf(codes[s], kmax)
        np.testing.assert_allclose(acf[s], a, rtol=0, atol=1e-12)
        want = A.detect_period(codes[s], kmax)
        near = np.any(np.abs(a[: max(want, kmax) if want == 0 else want] - 0.95) < 1e-9)
        assert period[s] == want or near, (s, period[s], want)


def test_zero_variance_and_constant():
    c = torch.full((2, 100), 5, dtype=torch.int32, device="cuda")
    p, a = bocd.detect_period(c, 10, with_acf=True)
    assert p.tolist() == [-1, -1] and not a.any()  # the zero-variance flag


def test_insufficient_data_is_an_error():
    c = torch.arange(40, dtype=torch.int32, device="cuda").view(2, 20)
    with pytest.raises(bocd.N.FalconError) as ei:
        bocd.detect_period(c, 11)  # |codes| < 2 k_max
    assert ei.value.code == bocd.N.FALCON_EINVAL


def test_iteration_times_match_oracle():
    rng = np.random.default_rng(3)
    S, n = 9, 1001
    ts = np.cumsum(rng.uniform(0.01, 0.2, size=(S, n)), axis=1)
    periods = np.array([0, 1, 2, 3, 4, 7, 100, 1000, 1001], dtype=np.int32)
    out, cnt = bocd.iteration_times(torch.from_numpy(ts).cuda(), torch.from_numpy(periods).cuda())
    out, cnt = out.cpu().numpy(), cnt.cpu().numpy()
    for s in range(S):
        want = A.iteration_times(ts[s], periods[s])
        assert cnt[s] == len(want)
        assert np.array_equal(out[s, : cnt[s]], want)


def test_tracking_chain_end_to_end():
    """per-rank NCCL call codes with a recurring period and timestamps whose
    iteration time rises by 30% over iterations 300-500 on rank 1 only."""
    rng = np.random.default_rng(2410_12588)
    S, L = 4, 9 * 801  # the same number of calls per rank: >= 800 iterations at every period
    Ps = [4, 6, 5, 9]
    codes, ts = [], []
    for s, P in enumerate(Ps):
        n_iter = L // P + 1
        blk = rng.integers(1, 9, size=P)
        c = np.tile(blk, n_iter)
        dur = 1.0 + 0.01 * rng.standard_normal(n_iter)
        if s == 1:
            dur[300:501] *= 1.3
        # calls spread uniformly within each iteration
        t = np.concatenate([[0.0], np.cumsum(np.repeat(dur / P, P))])[: len(c)]
        codes.append(c)
        ts.append(t)
    codes_d = torch.from_numpy(np.stack([c[:L] for c in codes]).astype(np.int32)).cuda()
    ts_d = torch.from_numpy(np.stack([t[:L] for t in ts])).cuda()
    period = bocd.detect_period(codes_d, 64)
    assert period.cpu().tolist() == Ps
    it, cnt = bocd.iteration_times(ts_d, period)
    T = int(cnt.min())
    x = it[:, :T].contiguous()
    b = bocd.BocdBatch(S, R=256, hazard=1 / 250, prior_first_obs=True, prior_cov=0.05, event_mask=3,
                       event_capacity=256)
    b.update_chunk(x)
    ev, _ = b.changepoints()
    b.close()
    verified = bocd.verify_changepoints(x, ev)
    fs = bocd.pair_failslow(verified)
    assert len(fs) == 1 and fs[0]["series"] == 1, fs
    assert 300 <= fs[0]["onset"] <= 305 and 500 <= fs[0]["recovery"] <= 506
    assert fs[0]["severity"] == pytest.approx(1.3, rel=0.03)
