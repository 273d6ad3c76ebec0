"""N2 ACF period detection throughput (falcon_detect_period) on one B200: one JSON line per
shape.  Work = sum_{k=1}^{k_max} (L - k) fp64 FMAs per rank (the lag sums of P:718-745);
reported against the FP64 pipe (148 SMs x 64 DFMA/clk x 1965 MHz) and the measured DFMA rate.
(Correctness: tests/test_gpu_acf.py against the oracle.)

    python tools/bench_acf.py
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_12588_b200 import bocd  # noqa: E402

PEAK = 148 * 64 * 1965e6
MEASURED = 1.7085e13


def run(S, L, kmax, reps=20):
    rng = np.random.default_rng(S + L)
    P = rng.integers(3, 13, size=S)
    # blocks of distinct codes: the smallest period is the block length
    codes = np.stack([np.tile(rng.permutation(20)[:p] + 1, L // p + 1)[:L] for p in P]).astype(np.int32)
    c = torch.from_numpy(codes).cuda()
    for _ in range(3):
        bocd.detect_period(c, kmax)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        bocd.detect_period(c, kmax)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    fma = S * sum(L - k for k in range(1, kmax + 1))

    return {"ranks": S, "L": L, "k_max": kmax, "ms": ms, "fma_per_s": fma / (ms * 1e-3),
            "frac_fp64_nominal": fma / (ms * 1e-3) / PEAK, "frac_fp64_measured": fma / (ms * 1e-3) / MEASURED}


if __name__ == "__main__":
    for S, L, kmax in ((1024, 4096, 256), (4096, 4096, 256), (1024, 8192, 1024), (10240, 2048, 64)):
        print(json.dumps(run(S, L, kmax)), flush=True)
