"""fp64 CPU oracle for batched BOCD — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_2410_12588_b200``) never imports it, and the C source
(``oracle/bocd_oracle.c``) shares no code with the CUDA path.

The arithmetic lives in ``bocd_oracle.c`` (textbook recursion of PAPER.md
Appendix A; see that file's header for the per-step citations).
This module only builds the shared object with gcc and marshals numpy arrays.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bocd_oracle.c")
_LIB = os.path.join(_HERE, "liboracle_bocd.so")

TRUNC_MERGE = 0
TRUNC_DROP = 1
EV_PROB = 1
EV_MAPRESET = 2


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2, OpenMP, no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-D_GNU_SOURCE", "-ffp-contract=off", "-fopenmp",
               "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


class _Params(ctypes.Structure):
    _fields_ = [("R", ctypes.c_int32), ("hazard", ctypes.c_double), ("kappa0", ctypes.c_double),
                ("alpha0", ctypes.c_double), ("threshold", ctypes.c_double),
                ("trunc_mode", ctypes.c_int32), ("prior_first_obs", ctypes.c_int32),
                ("prior_cov", ctypes.c_double)]


_P = ctypes.c_void_p


class _Outputs(ctypes.Structure):
    _fields_ = [(n, _P) for n in ("log_z", "p_new", "margin", "map_rl", "cp_index", "flags",
                                  "logR_traj", "logR_final", "mu_final", "beta_final")]


_lib = None


def _load():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.oracle_bocd_run.restype = ctypes.c_int
        _lib.oracle_bocd_run.argtypes = [ctypes.POINTER(_Params), _P, ctypes.c_int64,
                                         ctypes.c_int64, ctypes.c_int64, _P, ctypes.c_double,
                                         _P, ctypes.c_double, ctypes.POINTER(_Outputs),
                                         ctypes.c_int]
        _lib.oracle_student_t_logpdf.restype = ctypes.c_double
        _lib.oracle_student_t_logpdf.argtypes = [ctypes.c_double] * 5
        _lib.oracle_nig_update.restype = None
        _lib.oracle_nig_update.argtypes = [ctypes.c_double] + [ctypes.POINTER(ctypes.c_double)] * 4
        _lib.oracle_max_threads.restype = ctypes.c_int
    return _lib


def student_t_logpdf(x, mu, kappa, alpha, beta) -> float:
    """O2: log St(x; 2 alpha, mu, beta (kappa+1)/(alpha kappa))."""
    return _load().oracle_student_t_logpdf(float(x), float(mu), float(kappa), float(alpha),
                                           float(beta))


def nig_update(x, mu, kappa, alpha, beta):
    """O7: one conjugate update; returns (mu', kappa', alpha', beta')."""
    m, k, a, b = (ctypes.c_double(v) for v in (mu, kappa, alpha, beta))
    _load().oracle_nig_update(float(x), ctypes.byref(m), ctypes.byref(k), ctypes.byref(a),
                              ctypes.byref(b))
    return m.value, k.value, a.value, b.value


def max_threads() -> int:
    return int(_load().oracle_max_threads())


@dataclass
class OracleResult:
    log_z: np.ndarray
    p_new: np.ndarray
    margin: np.ndarray
    map_rl: np.ndarray
    cp_index: np.ndarray
    flags: np.ndarray
    logR_final: np.ndarray
    mu_final: np.ndarray
    beta_final: np.ndarray
    logR_traj: np.ndarray | None

    def events(self, event_mask: int = EV_PROB):
        """O9: (series, t, cp_index, flags, p_new) for t >= 1 with flags & mask, (series, t) order."""
        s_idx, t_idx = np.nonzero((self.flags & event_mask) != 0)
        return [(int(s), int(t), int(self.cp_index[s, t]), int(self.flags[s, t]),
                 float(self.p_new[s, t])) for s, t in zip(s_idx, t_idx)]


def run(x, R, hazard, kappa0=1.0, alpha0=1.0, mu0=None, beta0=None, threshold=0.9,
        trunc_mode=TRUNC_MERGE, prior_first_obs=False, prior_cov=0.05, traj=False,
        n_threads=0) -> OracleResult:
    """Run the oracle over x[S][T] (fp64).  mu0/beta0: scalar or per-series arrays."""
    x = np.ascontiguousarray(np.atleast_2d(np.asarray(x, dtype=np.float64)))
    S, T = x.shape
    p = _Params(int(R), float(hazard), float(kappa0), float(alpha0), float(threshold),
                int(trunc_mode), int(bool(prior_first_obs)), float(prior_cov))

    def per_series(v, default):
        if v is None:
            return None, default
        a = np.asarray(v, dtype=np.float64)
        if a.ndim == 0:
            return None, float(a)
        a = np.ascontiguousarray(a.reshape(S))
        return a, 0.0

    mu_arr, mu_sc = per_series(mu0, 0.0)
    be_arr, be_sc = per_series(beta0, 1.0)
    out = {
        "log_z": np.empty((S, T)), "p_new": np.empty((S, T)), "margin": np.empty((S, T)),
        "map_rl": np.empty((S, T), np.int32), "cp_index": np.empty((S, T), np.int64),
        "flags": np.empty((S, T), np.uint32), "logR_final": np.empty((S, R)),
        "mu_final": np.empty((S, R)), "beta_final": np.empty((S, R)),
        "logR_traj": np.empty((S, T, R)) if traj else None,
    }
    o = _Outputs(**{k: (v.ctypes.data if v is not None else None) for k, v in out.items()})
    rc = _load().oracle_bocd_run(
        ctypes.byref(p), x.ctypes.data if x.size else None, S, T, T,
        mu_arr.ctypes.data if mu_arr is not None else None, mu_sc,
        be_arr.ctypes.data if be_arr is not None else None, be_sc, ctypes.byref(o),
        int(n_threads))
    if rc == -1:
        raise FloatingPointError("oracle: non-finite observation (Q13)")
    if rc != 0:
        raise ValueError(f"oracle_bocd_run failed with code {rc}")
    return OracleResult(**out)
