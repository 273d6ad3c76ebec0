"""T2 — oracle invariants and hand-built examples.

* Normalisation: sum_r R_t(r) = 1 at every step.
* Change-point mass: untruncated and MERGE give R_t(0) = H exactly (the
  normaliser equals the change-point log-sum-exp); DROP gives R_t(0) >= H.
* The BASELINE.json configs[0] example (C1: 1.5x step at t=600, H = 1/250,
  R = 256): the only PROB event for t >= 1 is (t=600, r*=1, cp_index=600), in
  both modes, noise-free and with 2% log-normal noise; MERGE fires MAPRESET
  once, at t=600 (readings Q4, Q5, Q8).
* a constant stream never exceeds 0.9; a 1.0 -> 2.0 step at
  t=50 with sigma=0.01 exceeds 0.9 within 5 samples.
* Metamorphic: x*2^k with mu0*2^k and beta0*4^k, and x+c with mu0+c, leave the
  posterior unchanged; H -> 0 makes the MAP run length the longest run.
"""
import numpy as np
import pytest

from paper_2410_12588_b200 import tracegen


def _c1(sigma, mode, oracle_mod):
    cfg = tracegen.CONFIGS["C1"]
    spec = tracegen.make_spec(cfg, sigma=sigma)
    x = tracegen.generate(spec)
    return x, oracle_mod.run(x, cfg.R, cfg.hazard, cfg.kappa0, cfg.alpha0, prior_first_obs=True,
                             prior_cov=cfg.prior_cov, trunc_mode=mode, traj=True)


@pytest.mark.parametrize("mode", [0, 1])
def test_normalisation_and_cp_mass(oracle_mod, mode):
    rng = np.random.default_rng(5)
    x = np.exp(rng.normal(0, 0.2, (3, 400))) * np.where(np.arange(400) > 250, 1.7, 1.0)
    res = oracle_mod.run(x, 64, 0.01, 1.0, 1.0, prior_first_obs=True, prior_cov=0.2,
                         trunc_mode=mode, traj=True)
    P = np.exp(res.logR_traj)
    np.testing.assert_allclose(P.sum(axis=2), 1.0, rtol=0, atol=1e-12)
    if mode == oracle_mod.TRUNC_MERGE:
        np.testing.assert_allclose(P[:, :, 0], 0.01, rtol=1e-11)
    else:
        assert np.all(P[:, :, 0] >= 0.01 * (1 - 1e-12))
        assert np.any(P[:, 64:, 0] > 0.0101)  # slot R-1 holds mass once regimes outlast R


def test_untruncated_cp_mass(oracle_mod):
    rng = np.random.default_rng(6)
    x = rng.normal(1, 0.1, (2, 60))
    res = oracle_mod.run(x, 64, 0.03, 0.5, 2.0, mu0=1.0, beta0=0.05, trunc_mode=1, traj=True)
    np.testing.assert_allclose(np.exp(res.logR_traj[:, :, 0]), 0.03, rtol=1e-11)


@pytest.mark.parametrize("sigma", [0.0, 0.02])
@pytest.mark.parametrize("mode", [0, 1])
def test_c1_step_example(oracle_mod, sigma, mode):
    x, res = _c1(sigma, mode, oracle_mod)
    ev = res.events(oracle_mod.EV_PROB)
    assert [(e[1], e[2]) for e in ev] == [(600, 600)]
    assert res.map_rl[0, 600] == 1
    if mode == oracle_mod.TRUNC_MERGE:
        resets = [e[1] for e in res.events(oracle_mod.EV_MAPRESET)]
        assert resets == [600]
    assert res.flags[0, 0] == 0  # no events at t = 0 (Q8)


def test_spec_constant_stream(oracle_mod):
    x = np.ones((1, 300))
    res = oracle_mod.run(x, 128, 1e-3, 1.0, 1.0, prior_first_obs=True, prior_cov=0.05)
    assert np.all(res.p_new[0, 10:] < 0.9)
    assert res.events(oracle_mod.EV_PROB) == []


def test_spec_step_detected_within_5(oracle_mod):
    rng = np.random.default_rng(9)
    x = np.where(np.arange(120) < 50, 1.0, 2.0) + rng.normal(0, 0.01, 120)
    res = oracle_mod.run(x[None, :], 128, 1e-3, 1.0, 1.0, prior_first_obs=True, prior_cov=0.05)
    hits = np.nonzero(res.p_new[0, 1:] > 0.9)[0] + 1
    assert len(hits) >= 1 and 50 <= hits[0] <= 55


@pytest.mark.parametrize("mode", [0, 1])
def test_metamorphic_scale_and_shift(oracle_mod, mode):
    x, base = _c1(0.02, mode, oracle_mod)
    mu0 = x[0, 0]
    b0 = 1.0 * (0.05 * mu0) ** 2
    ref = oracle_mod.run(x, 256, 1 / 250, 1.0, 1.0, mu0, b0, trunc_mode=mode, traj=True)
    np.testing.assert_array_equal(ref.logR_traj, base.logR_traj)  # explicit prior == first-obs prior
    k = 5
    sc = oracle_mod.run(x * 2.0 ** k, 256, 1 / 250, 1.0, 1.0, mu0 * 2.0 ** k, b0 * 4.0 ** k,
                        trunc_mode=mode, traj=True)
    live = ref.logR_traj > -50
    assert np.max(np.abs(sc.logR_traj[live] - ref.logR_traj[live])) < 1e-11
    sh = oracle_mod.run(x + 3.0, 256, 1 / 250, 1.0, 1.0, mu0 + 3.0, b0, trunc_mode=mode, traj=True)
    assert np.max(np.abs(sh.logR_traj[live] - ref.logR_traj[live])) < 1e-9
    # the Student-t depends on the data only through differences: the log evidence shifts by
    # -T log 2^k under the scaling, and is unchanged under the shift
    np.testing.assert_allclose(sc.log_z.sum(), ref.log_z.sum() - x.shape[1] * k * np.log(2.0),
                               rtol=0, atol=1e-8)


def test_tiny_hazard_map_is_longest_run(oracle_mod):
    rng = np.random.default_rng(12)
    x = rng.normal(1, 0.1, (1, 40))
    res = oracle_mod.run(x, 64, 1e-12, 1.0, 1.0, mu0=1.0, beta0=0.01)
    np.testing.assert_array_equal(res.map_rl[0], np.arange(1, 41))
    np.testing.assert_array_equal(res.cp_index[0], 0)


@pytest.mark.parametrize("mode", [0, 1])
def test_minimal_R2(oracle_mod, mode):
    x = np.array([[1.0, 1.1, 0.9, 3.0, 3.1]])
    res = oracle_mod.run(x, 2, 0.1, 1.0, 1.0, mu0=1.0, beta0=0.01, trunc_mode=mode, traj=True)
    np.testing.assert_allclose(np.exp(res.logR_traj).sum(axis=2), 1.0, atol=1e-14)
    assert np.all(res.map_rl == 1)


def test_nonfinite_raises(oracle_mod):
    x = np.array([[1.0, np.nan, 1.0]])
    with pytest.raises(FloatingPointError):
        oracle_mod.run(x, 8, 0.1, mu0=1.0, beta0=0.1)
