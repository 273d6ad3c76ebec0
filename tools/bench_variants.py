"""Kernel time of one 1,000-step update_chunk for the kernel variants a user can land on:
the FULL kernels (power-of-two R = NT x J; a fractional 2 alpha0 adds one DADD per cell) and the
generic ones (any other R), C3-recipe data, device-resident, CUDA events.
One JSON line per case.

    python tools/bench_variants.py
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_12588_b200 import bocd, tracegen  # noqa: E402

CASES = [  # (R, alpha0, series)
    (1024, 1.0, 32768), (1024, 0.7, 32768), (1000, 1.0, 32768), (300, 1.0, 32768),
    (256, 1.0, 32768), (512, 1.0, 32768), (2048, 1.0, 16384), (4096, 1.0, 8192), (4096, 0.7, 8192),
]


def run(R, alpha0, S, T=1000, reps=3):
    cfg = tracegen.CONFIGS["C3"]
    spec = tracegen.make_spec(cfg, n_series=S)
    gen = bocd.DeviceTrace(spec, torch.device("cuda"))
    x = torch.empty((S, (reps + 2) * T), dtype=torch.float64, device="cuda")
    gen.generate(x, 0, 0)
    b = bocd.BocdBatch(S, R=R, hazard=cfg.hazard, alpha0=alpha0, prior_first_obs=True,
                       prior_cov=cfg.prior_cov, event_capacity=4096)
    for k in range(2):
        b.update_chunk(x[:, k * T:(k + 1) * T])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(2, reps + 2):
        b.update_chunk(x[:, k * T:(k + 1) * T])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    nt, j, spb = b.kernel_shape()
    b.changepoints()
    b.close()
    full = R == nt * j
    cells = S * T * R
    return {"R": R, "alpha0": alpha0, "series": S, "steps": T, "kernel": "FULL" if full else "generic",
            "shape": [nt, j, spb], "ms": ms, "ns_per_kcells": ms * 1e6 / (cells / 1e3),
            "series_steps_per_s": S * T / (ms * 1e-3)}


if __name__ == "__main__":
    for R, a0, S in CASES:
        print(json.dumps(run(R, a0, S)), flush=True)
