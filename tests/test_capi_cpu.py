"""C ABI checks that need no GPU: the library loads, exports every symbol the
headers declare, validates its arguments, refuses to run without a device (no
CPU fallback), and its per-run-length predictive constants are within 1 ulp of
50-digit mpmath (reading Q11; Student-t normaliser of the UPM predictive,
P:1333 / P:1345)."""
import ctypes
import math
import os
import re

import mpmath
import numpy as np
import pytest

from paper_2410_12588_b200 import _native as N
from paper_2410_12588_b200 import build as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    B.build()
    return N.lib()


def _declared():
    names = set()
    for h in ("falcon_bocd.h", "falcon_trace.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        names |= set(re.findall(r"^\s*(?:int|const char \*)\s*\**(falcon_\w+)\s*\(", src, re.M))
    return names


def test_exports_every_declared_symbol(L):
    decl = _declared()
    assert len(decl) >= 14
    for name in decl:
        assert hasattr(L, name), name
    assert set(N.EXPORTED) == decl
    assert L.falcon_bocd_abi_version() == 1


def test_config_defaults(L):
    c = N.Config()
    assert L.falcon_bocd_config_init(ctypes.byref(c)) == 0
    assert c.R == 1024 and c.hazard == 1 / 250 and c.threshold == 0.9
    assert c.trunc_mode == N.TRUNC_MERGE and c.event_mask == N.EV_PROB and c.event_capacity == 64


@pytest.mark.parametrize("field,val", [("R", 1), ("R", 5000), ("hazard", 0.0), ("hazard", 1.0),
                                       ("kappa0", 0.0), ("alpha0", -1.0), ("trunc_mode", 7),
                                       ("event_capacity", 0), ("n_series", 0),
                                       ("beta0_scalar", 0.0)])
def test_create_rejects_bad_config(L, field, val):
    c = N.Config()
    L.falcon_bocd_config_init(ctypes.byref(c))
    setattr(c, field, val)
    h = ctypes.c_void_p()
    assert L.falcon_bocd_create(ctypes.byref(c), ctypes.byref(h)) == N.FALCON_EINVAL
    assert not h.value
    assert L.falcon_bocd_last_error(None)


def test_no_cpu_fallback(L):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    c = N.Config()
    L.falcon_bocd_config_init(ctypes.byref(c))
    h = ctypes.c_void_p()
    rc = L.falcon_bocd_create(ctypes.byref(c), ctypes.byref(h))
    assert rc == N.FALCON_ECUDA and not h.value
    assert b"no CPU fallback" in L.falcon_bocd_last_error(None)


def test_null_handle_paths(L):
    n = ctypes.c_int64()
    assert L.falcon_bocd_destroy(None) == 0
    assert L.falcon_bocd_update_chunk(None, None, 0, 0, None, None) == N.FALCON_EINVAL
    assert L.falcon_bocd_changepoints(None, None, 0, ctypes.byref(n), None) == N.FALCON_EINVAL
    assert L.falcon_bocd_read_posterior(None, 0, 0, None, None, None, None) == N.FALCON_EINVAL


@pytest.mark.parametrize("R,kappa0,alpha0", [(4096, 1.0, 1.0), (512, 0.37, 2.25), (64, 5.0, 0.5)])
def test_predictive_constants_within_1ulp(L, R, kappa0, alpha0):
    out = [np.empty(R) for _ in range(4)]
    assert L.falcon_bocd_predictive_constants(R, kappa0, alpha0, *[o.ctypes.data for o in out]) == 0
    c, a, g, k1 = out
    mpmath.mp.dps = 50
    for r in list(range(0, 40)) + list(range(R - 40, R)) + list(range(40, R - 40, max(1, R // 64))):
        kap = mpmath.mpf(kappa0) + r
        alp = mpmath.mpf(alpha0) + mpmath.mpf(r) / 2
        cr = (mpmath.loggamma(alp + mpmath.mpf(1) / 2) - mpmath.loggamma(alp)
              - mpmath.log(2 * mpmath.pi * (kap + 1) / kap) / 2)
        for got, ref in ((c[r], cr), (a[r], alp), (g[r], kap / (2 * (kap + 1))), (k1[r], 1 / (kap + 1))):
            ref = float(ref)
            assert abs(got - ref) <= math.ulp(ref), (r, got, ref)


@pytest.mark.parametrize("R,kappa0,alpha0", [(4096, 1.0, 1.0), (1024, 0.37, 2.25)])
def test_predictive_constants_telescope_to_the_marginal(L, R, kappa0, alpha0):
    """The log-joint kernel (bocd_kernel.cuh) uses G_n = sum_{r<n} c_r: the product of the
    Student-t predictives' constants telescopes into the NIG marginal likelihood's constant
    lnGamma(alpha_n) - lnGamma(alpha0) + 1/2 ln(kappa0/kappa_n) - n/2 ln(2 pi) (closed form,
    50-digit mpmath)."""
    out = [np.empty(R) for _ in range(4)]
    assert L.falcon_bocd_predictive_constants(R, kappa0, alpha0, *[o.ctypes.data for o in out]) == 0
    c = out[0]
    G = np.cumsum(c)  # G[n-1] = sum_{r<n} c_r
    mpmath.mp.dps = 50
    for n in (1, 2, 3, 17, R // 2, R - 1, R):
        al = mpmath.mpf(alpha0) + mpmath.mpf(n) / 2
        ref = (mpmath.loggamma(al) - mpmath.loggamma(mpmath.mpf(alpha0))
               + mpmath.log(mpmath.mpf(kappa0) / (kappa0 + n)) / 2 - n * mpmath.log(2 * mpmath.pi) / 2)
        assert abs(G[n - 1] - float(ref)) <= 1e-12 * max(1.0, abs(float(ref))), (n, G[n - 1], float(ref))
