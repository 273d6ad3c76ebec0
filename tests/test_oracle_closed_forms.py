"""T0 — pins of the oracle's per-cell arithmetic against closed forms and library routines.

The oracle's NIG update (O7) and Student-t predictive (O2) are checked against
results that do NOT come from the oracle's own formulas:
  * the batch (closed-form) NIG posterior — the sequential update must reproduce it;
  * scipy.stats.t.logpdf (a library routine) and mpmath at 50 digits;
  * the nu = 1 (Cauchy) and nu = 2 special cases of the Student-t density;
  * the chain rule: the sum of sequential predictives equals the closed-form
    NIG marginal likelihood (a plausible error in either update or predictive
    — a dropped (kappa+1) factor, a wrong alpha increment — breaks it).
Reading Q1: the paper's UPM is a Gaussian with
unknown mean and variance under a NIG prior.
"""
import math

import mpmath
import numpy as np
import pytest
import scipy.stats

pytestmark = []


def nig_batch(x, mu0, k0, a0, b0):
    """Closed-form NIG posterior after n observations (textbook conjugate result)."""
    x = np.asarray(x, dtype=np.float64)
    n = len(x)
    xb = x.mean()
    kn = k0 + n
    mun = (k0 * mu0 + n * xb) / kn
    an = a0 + n / 2.0
    bn = b0 + 0.5 * np.sum((x - xb) ** 2) + k0 * n * (xb - mu0) ** 2 / (2.0 * kn)
    return mun, kn, an, bn


def log_marginal_mp(x, mu0, k0, a0, b0):
    """log p(x_1..n) = log G(a_n)/G(a0) + a0 log b0 - a_n log b_n + 1/2 log(k0/k_n) - n/2 log(2 pi)."""
    mpmath.mp.dps = 50
    xs = [mpmath.mpf(float(v)) for v in x]
    n = len(xs)
    mu0, k0, a0, b0 = (mpmath.mpf(float(v)) for v in (mu0, k0, a0, b0))
    xb = sum(xs) / n
    kn = k0 + n
    an = a0 + mpmath.mpf(n) / 2
    bn = b0 + sum((v - xb) ** 2 for v in xs) / 2 + k0 * n * (xb - mu0) ** 2 / (2 * kn)
    return (mpmath.loggamma(an) - mpmath.loggamma(a0) + a0 * mpmath.log(b0) - an * mpmath.log(bn)
            + mpmath.log(k0 / kn) / 2 - n * mpmath.log(2 * mpmath.pi) / 2)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_nig_sequential_equals_batch(oracle_mod, seed):
    rng = np.random.default_rng(seed)
    x = rng.normal(rng.uniform(-3, 3), rng.uniform(0.01, 2.0), size=200)
    mu0, k0, a0, b0 = rng.normal(), rng.uniform(0.1, 5), rng.uniform(0.5, 5), rng.uniform(0.01, 3)
    m, k, a, b = mu0, k0, a0, b0
    for n, xv in enumerate(x, start=1):
        m, k, a, b = oracle_mod.nig_update(xv, m, k, a, b)
        if n in (1, 2, 7, 50, 200):
            mb, kb, ab, bb = nig_batch(x[:n], mu0, k0, a0, b0)
            assert k == pytest.approx(kb, rel=1e-14)
            assert a == pytest.approx(ab, rel=1e-14)
            assert m == pytest.approx(mb, rel=1e-13, abs=1e-13)
            assert b == pytest.approx(bb, rel=1e-12)


@pytest.mark.parametrize("alpha", [0.5, 1.0, 2.5, 17.0, 128.0, 512.5, 2048.0])
def test_student_t_vs_scipy(oracle_mod, alpha):
    rng = np.random.default_rng(int(alpha * 10))
    for _ in range(20):
        x, mu = rng.normal(0, 3), rng.normal(0, 1)
        kappa, beta = rng.uniform(0.5, 3000), rng.uniform(1e-4, 50)
        scale = math.sqrt(beta * (kappa + 1) / (alpha * kappa))
        ref = scipy.stats.t.logpdf(x, 2 * alpha, loc=mu, scale=scale)
        got = oracle_mod.student_t_logpdf(x, mu, kappa, alpha, beta)
        assert got == pytest.approx(ref, rel=1e-12, abs=1e-12)


@pytest.mark.parametrize("alpha", [1.0, 40.5, 512.0, 2048.5])
def test_student_t_vs_mpmath_50_digits(oracle_mod, alpha):
    """Pins the lgamma difference D(alpha) = lgamma(alpha+1/2) - lgamma(alpha) at large alpha (Q11)."""
    mpmath.mp.dps = 50
    rng = np.random.default_rng(7)
    for _ in range(10):
        x, mu = rng.normal(1, 0.2), rng.normal(1, 0.01)
        kappa, beta = 2 * alpha - 1 + 1.0, rng.uniform(1e-3, 10)
        a, k, b = mpmath.mpf(alpha), mpmath.mpf(kappa), mpmath.mpf(beta)
        nu = 2 * a
        s2 = b * (k + 1) / (a * k)
        z2 = (mpmath.mpf(x) - mpmath.mpf(mu)) ** 2 / (nu * s2)
        ref = (mpmath.loggamma((nu + 1) / 2) - mpmath.loggamma(nu / 2)
               - mpmath.log(nu * mpmath.pi * s2) / 2 - (nu + 1) / 2 * mpmath.log1p(z2))
        got = oracle_mod.student_t_logpdf(x, mu, kappa, alpha, beta)
        assert abs(got - float(ref)) <= 2e-14 * max(1.0, abs(float(ref)))


def test_cauchy_special_case(oracle_mod):
    """alpha = 1/2 -> nu = 1: log f = -log(pi s (1 + z^2))."""
    rng = np.random.default_rng(3)
    for _ in range(50):
        x, mu, kappa, beta = rng.normal(0, 5), rng.normal(), rng.uniform(0.1, 10), rng.uniform(0.01, 5)
        s = math.sqrt(beta * (kappa + 1) / (0.5 * kappa))
        z = (x - mu) / s
        ref = -math.log(math.pi * s * (1 + z * z))
        assert oracle_mod.student_t_logpdf(x, mu, kappa, 0.5, beta) == pytest.approx(ref, rel=1e-13, abs=1e-13)


def test_nu2_special_case(oracle_mod):
    """alpha = 1 -> nu = 2: f(z) = (2 sqrt 2 s)^-1 (1 + z^2/2)^(-3/2)."""
    rng = np.random.default_rng(4)
    for _ in range(50):
        x, mu, kappa, beta = rng.normal(0, 5), rng.normal(), rng.uniform(0.1, 10), rng.uniform(0.01, 5)
        s = math.sqrt(beta * (kappa + 1) / kappa)
        z = (x - mu) / s
        ref = -math.log(2 * math.sqrt(2) * s) - 1.5 * math.log1p(z * z / 2)
        assert oracle_mod.student_t_logpdf(x, mu, kappa, 1.0, beta) == pytest.approx(ref, rel=1e-13, abs=1e-13)


@pytest.mark.parametrize("seed", [0, 1])
def test_chain_rule_equals_marginal_likelihood(oracle_mod, seed):
    rng = np.random.default_rng(100 + seed)
    x = rng.normal(rng.uniform(0.5, 2), rng.uniform(0.01, 0.5), size=60)
    mu0, k0, a0, b0 = float(x[0]), rng.uniform(0.2, 3), rng.uniform(0.5, 3), rng.uniform(0.001, 0.5)
    m, k, a, b = mu0, k0, a0, b0
    total = 0.0
    for xv in x:
        total += oracle_mod.student_t_logpdf(xv, m, k, a, b)
        m, k, a, b = oracle_mod.nig_update(xv, m, k, a, b)
    ref = float(log_marginal_mp(x, mu0, k0, a0, b0))
    assert total == pytest.approx(ref, rel=1e-12, abs=1e-11)
