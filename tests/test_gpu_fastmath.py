"""Accuracy of the kernels' branch-free fp64 log2 / exp2 (csrc/fastmath.cuh) vs numpy and
mpmath, through the falcon_bocd_debug_fastmath C-ABI hook.  The BOCD recursion (in base-2
units) uses log2 on the NIG scale beta' (> 0, normal) and exp2 on lp - M (<= ~0)."""
import ctypes
import math

import mpmath
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2410_12588_b200 import _native as N  # noqa: E402


def _probe(which, x):
    xd = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()
    out = torch.empty_like(xd)
    rc = N.lib().falcon_bocd_debug_fastmath(which, ctypes.c_void_p(xd.data_ptr()),
                                            ctypes.c_void_p(out.data_ptr()), xd.numel(),
                                            ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == 0
    return out.cpu().numpy()


def test_fast_log2_accuracy():
    rng = np.random.default_rng(0)
    x = np.concatenate([
        np.exp(rng.uniform(np.log(1e-300), np.log(1e300), 200000)),
        rng.uniform(0.5, 2.0, 200000),
        1.0 + rng.normal(0, 1e-6, 20000),
        np.array([1.0, 2.0, 0.5, 0.70703125, 1.4140625, 0.7070312499999999, 1.4140624999999998,
                  np.nextafter(1.0, 2), np.nextafter(1.0, 0), 2.2250738585072014e-308, 1.7e308]),
    ])
    got = _probe(0, x)
    ref = np.log2(x)
    ulp = np.spacing(np.abs(ref))
    err = np.abs(got - ref)
    # absolute accuracy is what the recursion needs (differences of logs); near x = 1 the
    # result is tiny and its own ulp is meaningless, so allow 4e-18 absolute there
    bad = err > 2.0 * ulp + 4e-18
    assert not np.any(bad), list(zip(x[bad][:5], got[bad][:5], ref[bad][:5]))
    mpmath.mp.dps = 40
    for v in x[::9973]:  # spot-check numpy itself against 40 digits
        r = float(mpmath.log(mpmath.mpf(float(v)), 2))
        assert abs(got[list(x).index(v)] - r) <= 2.0 * math.ulp(r) + 4e-18


def test_fast_exp2_accuracy():
    rng = np.random.default_rng(1)
    x = np.concatenate([-rng.exponential(5.0, 200000), rng.uniform(-1021, 0, 200000),
                        -rng.uniform(0, 1e-3, 20000), np.array([0.0, -0.0, 1e-12, -1e-300, -1021.0])])
    got = _probe(1, x)
    ref = np.exp2(x)
    err = np.abs(got - ref) / ref
    assert np.all(err <= 2.5e-16), float(err.max())


def test_fast_exp2_clamps_below():
    x = np.array([-np.inf, -1e300, -1022.0, -1074.5, -1e5])
    got = _probe(1, x)
    assert np.all(np.isfinite(got)) and np.all(got >= 0) and np.all(got < 1e-306)


@pytest.mark.parametrize("which,bound", [(2, 1.1e-15), (4, 2e-18)])
def test_cell_log2_accuracy(which, bound):
    """The cell loop's log2 (csrc/cellmath.cuh): 2^LB intervals + degree-3 Chebyshev fit (max
    |error| 1.0e-15 at LB = 8, which 2; 9.9e-19 at LB = 10, which 4), plus the rounding of
    k + l_i: an ABSOLUTE error (the recursion uses alpha * lg beta' against a per-cell offset)
    within bound + 2 ulp(max(|log2 x|, 1))."""
    rng = np.random.default_rng(2)
    x = np.concatenate([
        np.exp(rng.uniform(np.log(1e-300), np.log(1e300), 200000)),
        rng.uniform(0.5, 4.0, 200000),
        1.0 + rng.normal(0, 1e-6, 20000),
        np.array([1.0, 2.0, 0.5, np.nextafter(1.0, 2), np.nextafter(1.0, 0), np.nextafter(2.0, 0),
                  2.2250738585072014e-308, 1.7e308]),
    ])
    got = _probe(which, x)
    ref = np.log2(x)
    err = np.abs(got - ref)
    bad = err > bound + 2.0 * np.spacing(np.maximum(np.abs(ref), 1.0))
    assert not np.any(bad), list(zip(x[bad][:5], got[bad][:5], ref[bad][:5]))


def test_cell_exp2_accuracy_and_floor():
    """The cell loop's exp2 (256-entry table, degree-4 Chebyshev fit): relative error within
    2.5e-16 on (-1021, 30]; below 2^-1021 (dead cells, and the finite offset -2^20 that
    impossible cells carry) the result is floored into [2^-1022, 2^-1018): a dead cell then
    carries < 2^-1010 of a step's evidence."""
    rng = np.random.default_rng(3)
    x = np.concatenate([-rng.exponential(5.0, 200000), rng.uniform(-1020.9, 0, 200000),
                        rng.uniform(0, 30, 20000), np.array([0.0, -0.0, 1e-12, -1e-300, -1020.5])])
    got = _probe(3, x)
    ref = np.exp2(x)
    err = np.abs(got - ref) / ref
    assert np.all(err <= 2.5e-16), float(err.max())
    dead = _probe(3, np.array([-1021.5, -1e4, -2e6, -1048576.0 - 3000.0]))
    assert np.all(dead >= 2.0 ** -1022) and np.all(dead < 2.0 ** -1018), dead
