"""B200-native batched BOCD — the data-parallel hot path of Falcon-Detect (arXiv 2410.12588).

Public API (thin bindings over libfalcon_bocd.so, see include/falcon_bocd.h):
    BocdBatch            falcon_bocd_create / _update_chunk(_host) / _changepoints /
                         _read_posterior / _destroy
    predictive_constants host-side per-run-length constant table
    DeviceTrace          device twin of the synthetic trace generator (falcon_trace_generate)
    distributed          series sharding + final NCCL allgather of change points
"""
from ._native import (EV_MAPRESET, EV_PROB, TRUNC_DROP, TRUNC_MERGE, FalconError,  # noqa: F401
                      LIB_PATH)

__all__ = ["BocdBatch", "predictive_constants", "DeviceTrace", "FalconError", "EV_PROB",
           "EV_MAPRESET", "TRUNC_MERGE", "TRUNC_DROP"]


def __getattr__(name):
    if name in ("BocdBatch", "predictive_constants", "DeviceTrace", "EVENT_DTYPE"):
        from . import bocd
        return getattr(bocd, name)
    raise AttributeError(name)
