"""Long-horizon precision of the resident kernel (R = 1024, MERGE, the C3 recipe) over
1,000,000 steps: the recursion of PAPER.md App. A is carried step after step
(P:1340-1348), and the online mode (BASELINE.json configs[4]) has no end, so any error
the kernel carries forward (the MERGE bucket's chain of merged masses, the frame) must not
drift toward the 1e-9 budget.  8 series x 1e6 steps through 10,000-step calls; the oracle
(fp64, textbook recursion) runs on the same bytes.  Checked: log Z_t and p_new at every
step, MAP outside exempt steps, the final log posterior; the per-100k-step maximum
|dlog Z| (the drift curve) goes to profiles/ when LONGHORIZON_OUT is set.
"""
import json
import os

import numpy as np
import pytest

from tests import parity

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2410_12588_b200 import bocd, tracegen  # noqa: E402

T_LONG = 1_000_000


def test_million_step_drift(oracle_mod):
    cfg = tracegen.CONFIGS["C3"]
    S, chunk = 8, 10_000
    spec = tracegen.make_spec(cfg, n_series=S, T=T_LONG)
    dt = bocd.DeviceTrace(spec, "cuda")
    b = bocd.BocdBatch(S, R=cfg.R, hazard=cfg.hazard, prior_first_obs=True, prior_cov=cfg.prior_cov,
                       event_mask=3, event_capacity=1 << 14)
    xs = torch.empty((S, chunk), dtype=torch.float64, device="cuda")
    x = np.empty((S, T_LONG))
    m = np.empty((S, T_LONG), np.int32)
    p = np.empty((S, T_LONG))
    z = np.empty((S, T_LONG))
    for t0 in range(0, T_LONG, chunk):
        dt.generate(xs, 0, t0)
        x[:, t0:t0 + chunk] = xs.cpu().numpy()
        mm, pp, zz = b.update_chunk(xs, outputs=True)
        m[:, t0:t0 + chunk] = mm.cpu().numpy()
        p[:, t0:t0 + chunk] = pp.cpu().numpy()
        z[:, t0:t0 + chunk] = zz.cpu().numpy()
    logR = b.read_posterior()[0].cpu().numpy()
    b.close()
    res = oracle_mod.run(x, cfg.R, cfg.hazard, prior_first_obs=True, prior_cov=cfg.prior_cov)
    dz = np.abs(z - res.log_z)
    curve = [float(dz[:, k:k + 100_000].max()) for k in range(0, T_LONG, 100_000)]
    dR = parity.compare_logR(logR, res.logR_final)
    st = parity.compare_steps(m, p, z, res, cfg.threshold)
    st.update(max_dlogR_final=dR, dlogz_per_100k=curve)
    parity.record(f"C3 recipe {S} x {T_LONG} steps, R=1024 MERGE", st)
    if os.environ.get("LONGHORIZON_OUT"):
        with open(os.environ["LONGHORIZON_OUT"], "w") as f:
            json.dump({"series": S, "steps": T_LONG, "R": cfg.R, "mode": "merge", "chunk": chunk,
                       "max_dlogz_per_100k_steps": curve, "max_dlogR_final": dR,
                       "max_dpnew": st["max_dpnew"], "exempt_steps": st["exempt_steps"]}, f, indent=1)
    # no trend toward the budget: the last 100k steps are within 10x of the first 100k and
    # well below 1e-9
    assert max(curve) < 1e-10
