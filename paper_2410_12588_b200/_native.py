"""ctypes view of libfalcon_bocd.so (include/falcon_bocd.h, include/falcon_trace.h).

Argument marshalling only.  Loading fails loudly if the shared object has not
been built: there is no CPU fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# FALCON_BOCD_LIB: load an alternative build of the same library (A/B tuning runs only)
LIB_PATH = os.environ.get("FALCON_BOCD_LIB") or os.path.join(HERE, "libfalcon_bocd.so")

FALCON_OK = 0
FALCON_WARN_EVENTS_DROPPED = 1
FALCON_EINVAL = -1
FALCON_ECUDA = -2
FALCON_ENOMEM = -3
FALCON_ENONFINITE = -4
FALCON_ESTATE = -5
TRUNC_MERGE = 0
TRUNC_DROP = 1
EV_PROB = 1
EV_MAPRESET = 2

_P = ctypes.c_void_p
_i32, _i64, _u32, _f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_double


class Config(ctypes.Structure):
    _fields_ = [("n_series", _i64), ("R", _i32), ("hazard", _f64), ("kappa0", _f64),
                ("alpha0", _f64), ("mu0", _P), ("mu0_scalar", _f64), ("beta0", _P),
                ("beta0_scalar", _f64), ("prior_first_obs", _i32), ("prior_cov", _f64),
                ("threshold", _f64), ("trunc_mode", _i32), ("event_mask", _u32),
                ("event_capacity", _i32), ("device", _i32), ("series_base", _i64)]


class Event(ctypes.Structure):
    _fields_ = [("series", _i64), ("t", _i64), ("cp_index", _i64), ("flags", _u32),
                ("reserved", _u32), ("p_new", _f64)]


class StepOut(ctypes.Structure):
    _fields_ = [("map_rl", _P), ("p_new", _P), ("log_z", _P), ("ld", _i64)]


class TraceSpecC(ctypes.Structure):
    _fields_ = [("seed", ctypes.c_uint64), ("n_series", _i64), ("gamma", _f64), ("b", _P),
                ("sigma", _P), ("ep_off", _P), ("ep_start", _P), ("ep_end", _P), ("ep_logsev", _P)]


class FalconError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"falcon_bocd error {code}: {msg}")
        self.code = code


_lib = None


def lib():
    """The loaded shared object (raises if it is missing)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built; run `python -m paper_2410_12588_b200.build` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    H = _P
    sig = {
        "falcon_bocd_abi_version": (ctypes.c_int, []),
        "falcon_bocd_config_init": (ctypes.c_int, [ctypes.POINTER(Config)]),
        "falcon_bocd_create": (ctypes.c_int, [ctypes.POINTER(Config), ctypes.POINTER(H)]),
        "falcon_bocd_update_chunk": (ctypes.c_int, [H, _P, _i64, _i64, ctypes.POINTER(StepOut), _P]),
        "falcon_bocd_update_chunk_host": (ctypes.c_int, [H, _P, _i64, _i64, ctypes.POINTER(StepOut), _P]),
        "falcon_bocd_changepoints": (ctypes.c_int, [H, _P, _i64, ctypes.POINTER(_i64), _P]),
        "falcon_bocd_changepoints_async": (ctypes.c_int, [H, _P, _i64, _P, _P]),
        "falcon_bocd_pending_events": (ctypes.c_int, [H, ctypes.POINTER(_i64), _P]),
        "falcon_bocd_read_posterior": (ctypes.c_int, [H, _i64, _i64, _P, _P, _P, _P]),
        "falcon_bocd_steps": (ctypes.c_int, [H, ctypes.POINTER(_i64)]),
        "falcon_bocd_set_schedule": (ctypes.c_int, [H, _i32]),
        "falcon_bocd_kernel_shape": (ctypes.c_int, [H, ctypes.POINTER(_i32), ctypes.POINTER(_i32),
                                                    ctypes.POINTER(_i32)]),
        "falcon_bocd_destroy": (ctypes.c_int, [H]),
        "falcon_bocd_last_error": (ctypes.c_char_p, [H]),
        "falcon_bocd_predictive_constants": (ctypes.c_int, [_i32, _f64, _f64, _P, _P, _P, _P]),
        "falcon_trace_generate": (ctypes.c_int, [ctypes.POINTER(TraceSpecC), _P, _i64, _i64, _i64,
                                                 _i64, _i64, _P]),
        "falcon_bocd_debug_fastmath": (ctypes.c_int, [_i32, _P, _P, _i64, _P]),
        "falcon_verify_changepoints": (ctypes.c_int, [_P, _i64, _i64, _i64, _i64, _i64, _P, _i64, _i32,
                                                      _f64, _P, _P]),
        "falcon_pair_failslow": (ctypes.c_int, [_P, _i64, _P, _i64, ctypes.POINTER(_i64), _P]),
        "falcon_classify_groups": (ctypes.c_int, [_P, _i64, _i32, _i64, _f64, _P, _P, _P]),
        "falcon_detect_period": (ctypes.c_int, [_P, _i64, _i32, _i64, _i32, _f64, _P, _P, _P]),
        "falcon_iteration_times": (ctypes.c_int, [_P, _i64, _i32, _i64, _P, _P, _i64, _P, _P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


EXPORTED = ["falcon_bocd_abi_version", "falcon_bocd_config_init", "falcon_bocd_create",
            "falcon_bocd_update_chunk", "falcon_bocd_update_chunk_host", "falcon_bocd_changepoints", "falcon_bocd_changepoints_async",
            "falcon_bocd_pending_events", "falcon_bocd_read_posterior", "falcon_bocd_steps",
            "falcon_bocd_set_schedule",
            "falcon_bocd_kernel_shape", "falcon_bocd_destroy", "falcon_bocd_last_error",
            "falcon_bocd_predictive_constants", "falcon_trace_generate", "falcon_bocd_debug_fastmath",
            "falcon_verify_changepoints", "falcon_pair_failslow", "falcon_classify_groups",
            "falcon_detect_period", "falcon_iteration_times"]
CP_JITTER, CP_DEGRADE, CP_RECOVER, CP_INSUFFICIENT = 0, 1, 2, 3


def check(code, handle=None):
    if code < 0:
        msg = lib().falcon_bocd_last_error(handle)
        raise FalconError(code, msg.decode() if msg else "")
    return code
