"""Secondary measurements for BASELINE.md's results table (the bench.py line is the C3
headline).  Device-resident inputs, CUDA-event timing, one GPU:
  C2  1,024 series x (10 x 1,000) steps, R = 512
  C4  12,500 series (one rank's share of 100,000 on 8 GPUs) x (5 x 1,000) steps, R = 4096
  C5  streaming: 10,240 series, one observation per call (T = 1), R = 1024:
      per-call device latency and sustained series*steps/s over 2,000 back-to-back calls
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_12588_b200 import bocd, tracegen  # noqa: E402


def chunked(name, S, chunk, steps, warm=2):
    cfg = tracegen.CONFIGS[name]
    spec = tracegen.make_spec(cfg, n_series=S)
    dt = bocd.DeviceTrace(spec, "cuda")
    x = torch.empty((S, (steps + warm) * chunk), dtype=torch.float64, device="cuda")
    dt.generate(x, 0, 0)
    b = bocd.BocdBatch(S, R=cfg.R, hazard=cfg.hazard, prior_first_obs=True, prior_cov=cfg.prior_cov,
                       event_capacity=512)
    for k in range(warm):
        b.update_chunk(x[:, k * chunk:(k + 1) * chunk])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(warm, warm + steps):
        b.update_chunk(x[:, k * chunk:(k + 1) * chunk])
    ev, dropped = b.changepoints()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    nt, j, spb = b.kernel_shape()
    b.close()
    return {"config": name, "series": S, "R": cfg.R, "steps": steps * chunk, "ms": ms,
            "series_steps_per_s": S * steps * chunk / (ms * 1e-3), "events": int(len(ev)),
            "kernel_shape": [nt, j, spb]}


def streaming(S=10240, calls=2000, warm=200):
    cfg = tracegen.CONFIGS["C5"]
    spec = tracegen.make_spec(cfg, n_series=S)
    dt = bocd.DeviceTrace(spec, "cuda")
    x = torch.empty((S, calls + warm), dtype=torch.float64, device="cuda")
    dt.generate(x, 0, 0)
    xc = x.t().contiguous().t()  # column-major copy: column k is contiguous? (use row stride)
    b = bocd.BocdBatch(S, R=1024, hazard=cfg.hazard, prior_first_obs=True, prior_cov=cfg.prior_cov,
                       event_capacity=512)
    for k in range(warm):
        b.update_chunk(x[:, k:k + 1])
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(calls + 1)]
    ev[0].record()
    for k in range(calls):
        b.update_chunk(x[:, warm + k:warm + k + 1])
        ev[k + 1].record()
    torch.cuda.synchronize()
    lat = sorted(ev[k].elapsed_time(ev[k + 1]) for k in range(calls))
    tot = ev[0].elapsed_time(ev[-1])
    b.close()
    del xc
    return {"config": "C5", "series": S, "R": 1024, "calls": calls,
            "per_call_ms_median": lat[len(lat) // 2], "per_call_ms_p99": lat[int(0.99 * len(lat))],
            "series_steps_per_s": S * calls / (tot * 1e-3),
            "hbm_bytes_per_call": S * 1024 * 24 * 2 + S * 8}


if __name__ == "__main__":
    out = [chunked("C2", 1024, 1000, 10), chunked("C4", 12500, 1000, 5), streaming()]
    for o in out:
        print(json.dumps(o), flush=True)
