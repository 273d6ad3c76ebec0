"""Throughput of the §8 "next" rows N1 (change-point verification, fail-slow pairing) and N4
(suspicious-group classification) on one B200, device-resident inputs, CUDA events around
the C-ABI calls (no host copies inside the timed region except pair_failslow's documented
count read-back).  One JSON line per shape, with the algorithmic bytes per call against the
measured HBM copy peak (MEASURED_PEAKS.json).  Correctness: tests/test_gpu_verify.py and
tests/test_gpu_groups.py against the oracle.

    python tools/bench_next.py
"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2410_12588_b200 import _native as N  # noqa: E402
from paper_2410_12588_b200 import bocd  # noqa: E402

try:
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        HBM = float(json.load(f)["hbm_gbs"]) * 1e9
except (OSError, KeyError, ValueError):
    HBM = 7.7e12  # the profiling guide's nominal figure


def _time(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def verify(S, T, n_ev, window=20, reps=20):
    """N1 V1-V3: per event 2 x window fp64 reads + a 40-B event record in, a 56-B record out."""
    rng = np.random.default_rng(n_ev)
    x = torch.from_numpy(rng.lognormal(0.0, 0.1, size=(S, T))).cuda()
    ev = np.zeros(n_ev, dtype=bocd.EVENT_DTYPE)
    ev["series"] = np.sort(rng.integers(0, S, n_ev))
    ev["cp_index"] = rng.integers(window, T - window, n_ev)
    ev["t"] = ev["cp_index"] + 5
    ev_d = torch.from_numpy(ev.view(np.uint8).reshape(n_ev, -1)).cuda()
    out_d = torch.empty((n_ev, bocd.VERIFIED_DTYPE.itemsize), dtype=torch.uint8, device="cuda")
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    lib = N.lib()

    def call():
        N.check(lib.falcon_verify_changepoints(ctypes.c_void_p(x.data_ptr()), T, S, 0, 0, T,
                                               ctypes.c_void_p(ev_d.data_ptr()), n_ev, window, 0.10,
                                               ctypes.c_void_p(out_d.data_ptr()), st))

    ms = _time(call, reps)
    byt = n_ev * (2 * window * 8 + bocd.EVENT_DTYPE.itemsize + bocd.VERIFIED_DTYPE.itemsize)
    return {"row": "N1 verify", "series": S, "T": T, "events": n_ev, "window": window, "ms": ms,
            "events_per_s": n_ev / (ms * 1e-3), "algorithmic_gbs": byt / (ms * 1e-3) / 1e9,
            "frac_hbm": byt / (ms * 1e-3) / HBM}


def pair(S, n, reps=20):
    """N1 V4: per verified record 56 B in; fail-slow events out (32 B each)."""
    rng = np.random.default_rng(n)
    v = np.zeros(n, dtype=bocd.VERIFIED_DTYPE)
    v["series"] = np.sort(rng.integers(0, S, n))
    v["t"] = np.arange(n)  # increasing within every series
    v["cp_index"] = v["t"] - 3
    v["status"] = rng.integers(0, 3, n)
    v["mean_before"] = 1.0
    v["mean_after"] = rng.uniform(0.5, 2.0, n)
    v_d = torch.from_numpy(v.view(np.uint8).reshape(n, -1)).cuda()
    cap = n
    out_d = torch.empty((cap, bocd.FAILSLOW_DTYPE.itemsize), dtype=torch.uint8, device="cuda")
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    n_out = ctypes.c_int64()
    lib = N.lib()

    def call():
        N.check(lib.falcon_pair_failslow(ctypes.c_void_p(v_d.data_ptr()), n, ctypes.c_void_p(out_d.data_ptr()),
                                         cap, ctypes.byref(n_out), st))

    ms = _time(call, reps)
    byt = n * bocd.VERIFIED_DTYPE.itemsize + n_out.value * bocd.FAILSLOW_DTYPE.itemsize
    return {"row": "N1 pair_failslow", "series": S, "records": n, "failslow_events": n_out.value, "ms": ms,
            "records_per_s": n / (ms * 1e-3), "algorithmic_gbs": byt / (ms * 1e-3) / 1e9,
            "frac_hbm": byt / (ms * 1e-3) / HBM, "note": "includes the documented host read-back of the count"}


def groups(B, G, reps=20):
    """N4: per batch G fp64 in, G flags + the median out; a shared-memory bitonic sort per batch."""
    rng = np.random.default_rng(B * G)
    t = torch.from_numpy(rng.lognormal(0.0, 0.2, size=(B, G))).cuda()
    ms = _time(lambda: bocd.classify_groups(t), reps)
    byt = B * G * 9 + B * 8
    return {"row": "N4 classify_groups", "batches": B, "groups": G, "ms": ms,
            "batches_per_s": B / (ms * 1e-3), "algorithmic_gbs": byt / (ms * 1e-3) / 1e9,
            "frac_hbm": byt / (ms * 1e-3) / HBM}


if __name__ == "__main__":
    for S, T, n in ((32768, 1000, 100_000), (32768, 1000, 1_000_000)):
        print(json.dumps(verify(S, T, n)), flush=True)
    for S, n in ((32768, 100_000), (32768, 1_000_000)):
        print(json.dumps(pair(S, n)), flush=True)
    for B, G in ((100_000, 64), (4096, 1024), (512, 8192)):
        print(json.dumps(groups(B, G)), flush=True)
