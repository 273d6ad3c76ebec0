"""T1 — the oracle's whole recursion (O1-O7) vs brute-force enumeration of segmentations.

For t <= 11 every boundary pattern is enumerated in mpmath (tests/bruteforce.py),
for R in {3, 4, 5, 16}, both truncation modes (reading Q6), several priors.  A
mistake anywhere in the recursion — a wrong slot shift, a missing hazard term,
a wrong merge of the bucket, stats that do not follow their run length — moves
the posterior by far more than the 1e-12 tolerance.  The cumulative
normaliser sum_t log Z_t must equal the brute-force log evidence.
"""
import numpy as np
import pytest

from tests import bruteforce

CASES = []
for R in (3, 4, 5, 16):
    for mode in ("drop", "merge"):
        CASES.append((R, mode, 0))
CASES += [(4, "drop", 1), (4, "merge", 1), (3, "merge", 2), (5, "drop", 2)]


def _data(variant):
    if variant == 0:  # SURVEY App. A shape: 6 points near 1.0, then 5 near 1.5
        rng = np.random.default_rng(11)
        x = np.concatenate([rng.normal(1.0, 0.05, 6), rng.normal(1.5, 0.05, 5)])
        return x, dict(mu0=1.0, k0=1.0, a0=1.0, b0=0.01, H=0.2)
    rng = np.random.default_rng(100 + variant)
    x = rng.normal(0, 1, 11) * rng.uniform(0.1, 2) + np.repeat(rng.normal(0, 2, 3), [4, 4, 3])
    return x, dict(mu0=rng.normal(), k0=rng.uniform(0.2, 3), a0=rng.uniform(0.5, 3),
                   b0=rng.uniform(0.05, 2), H=rng.uniform(0.05, 0.5))


@pytest.mark.parametrize("R,mode,variant", CASES)
def test_recursion_equals_enumeration(oracle_mod, R, mode, variant):
    x, pr = _data(variant)
    ref, evid = bruteforce.posterior(x, R, pr["H"], pr["mu0"], pr["k0"], pr["a0"], pr["b0"], mode)
    res = oracle_mod.run(x[None, :], R, pr["H"], pr["k0"], pr["a0"], pr["mu0"], pr["b0"],
                         trunc_mode=oracle_mod.TRUNC_DROP if mode == "drop" else oracle_mod.TRUNC_MERGE,
                         traj=True)
    got = res.logR_traj[0]
    for t in range(len(x)):
        for r in range(R):
            a, b = got[t, r], ref[t][r]
            if b == float("-inf"):
                assert a == float("-inf"), (t, r, a)
            else:
                assert abs(a - b) < 1e-12, (t, r, a, b)
    cum = np.cumsum(res.log_z[0])
    np.testing.assert_allclose(cum, evid, rtol=0, atol=1e-11)
