"""Parity at BASELINE.json full sizes, in the launch configuration bench.py times, on sampled
outputs the oracle can compute (whole series, all steps) plus size-independent properties.

C2: 1,024 series x 10,000 steps (R=512) — 6 sampled series checked step by step.
C3: 32,768 series x 20,000 steps (R=1024, bench chunking: 1,000-step calls) — 4 sampled
    series checked against the oracle over all 20,000 steps; the event stream of every
    series is checked for the invariants t >= 1, cp_index <= t, p_new > 0.9; and the full
    C3 length, 100,000 steps (512 series, 2 sampled), where errors carried by the MERGE
    bucket would show.
"""
import numpy as np
import pytest

from tests import parity

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2410_12588_b200 import bocd, tracegen  # noqa: E402


def _run_full(cfg, S, T, chunk, sample, mode=0, cap=256, outputs=True):
    spec = tracegen.make_spec(cfg, n_series=S)
    dt = bocd.DeviceTrace(spec, "cuda")
    b = bocd.BocdBatch(S, R=cfg.R, hazard=cfg.hazard, prior_first_obs=True, prior_cov=cfg.prior_cov,
                       trunc_mode=mode, event_mask=1, event_capacity=cap)
    xs = torch.empty((S, chunk), dtype=torch.float64, device="cuda")
    outs = {k: [] for k in ("map", "pnew", "logz")}
    xsample = []
    for t0 in range(0, T, chunk):
        dt.generate(xs, 0, t0)
        xsample.append(xs[sample].cpu().numpy())
        res = b.update_chunk(xs, outputs=outputs)
        if outputs:
            outs["map"].append(res[0][sample].cpu().numpy())
            outs["pnew"].append(res[1][sample].cpu().numpy())
            outs["logz"].append(res[2][sample].cpu().numpy())
    logR = b.read_posterior()[0][sample].cpu().numpy()
    ev, dropped = b.changepoints()
    b.close()
    return (np.concatenate(xsample, 1), {k: np.concatenate(v, 1) for k, v in outs.items() if v}, logR,
            ev, dropped)


@pytest.mark.parametrize("cfgname,S,T,chunk,sample,outputs", [
    ("C2", 1024, 10000, 2500, [0, 1, 511, 777, 1022, 1023], True),
    ("C3", 32768, 20000, 1000, [0, 12345, 20000, 32767], False),  # bench launch configuration
    ("C3", 32768, 6000, 1000, [3, 4097, 32766], True),
    ("C3", 512, 100000, 1000, [7, 300], True),  # the full C3 length (100,000 steps)
])
def test_full_size_sampled_parity(oracle_mod, cfgname, S, T, chunk, sample, outputs):
    cfg = tracegen.CONFIGS[cfgname]
    x, g, logR, ev, dropped = _run_full(cfg, S, T, chunk, sample, outputs=outputs)
    # the sampled inputs are the device generator's bytes: both sides see the same x
    res = oracle_mod.run(x, cfg.R, cfg.hazard, prior_first_obs=True, prior_cov=cfg.prior_cov)
    st = {}
    if outputs:
        st = parity.compare_steps(g["map"], g["pnew"], g["logz"], res, cfg.threshold)
    st["max_dlogR"] = parity.compare_logR(logR, res.logR_final)
    parity.record(f"{cfgname} full {S}x{T} sampled {sample} outputs={outputs}", st)
    assert not dropped
    assert np.all(ev["t"] >= 1) and np.all(ev["cp_index"] <= ev["t"]) and np.all(ev["p_new"] > 0.9)
    assert np.all(np.diff(ev["series"]) >= 0)
    # the sampled series' events equal the oracle's (outside exempt steps)
    ex = parity.exempt_steps(res.margin, res.p_new, cfg.threshold)
    for k, s in enumerate(sample):
        got = {(int(e["t"]), int(e["cp_index"])) for e in ev[ev["series"] == s] if not ex[k, int(e["t"])]}
        want = {(t, c) for (si, t, c, f, p) in res.events(1) if si == k and not ex[k, t]}
        assert got == want, (s, sorted(got ^ want)[:5])
