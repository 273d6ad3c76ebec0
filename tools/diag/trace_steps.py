"""Diagnostic (not a bench): CUDA timeline of the bench's per-step loop (update + async drain)
under torch.profiler, to find gaps between kernels.  Prints per-kernel start/duration (us).

    python tools/diag/trace_steps.py [C2|C3] [steps]
"""
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2410_12588_b200 import bocd, tracegen  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg = tracegen.CONFIGS[name]
S, C = cfg.n_series, 1000
x = torch.empty((S, (steps + 3) * C), dtype=torch.float64, device="cuda")
bocd.DeviceTrace(tracegen.make_spec(cfg), "cuda").generate(x, 0, 0)
b = bocd.BocdBatch(S, R=cfg.R, hazard=cfg.hazard, prior_first_obs=True, prior_cov=cfg.prior_cov, event_capacity=256)
for k in range(3):
    b.update_chunk(x[:, k * C:(k + 1) * C])
    b.changepoints_async(device_out=True).result()
b.reserve_events(2 * max(b._ev_hint, 1024), device_out=True)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    pending = None
    for k in range(3, 3 + steps):
        b.update_chunk(x[:, k * C:(k + 1) * C])
        t = b.changepoints_async(device_out=True)
        if pending is not None:
            pending.result()
        pending = t
    pending.result()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
prev_end = None
for e in ev:
    gap = (e.time_range.start - prev_end) if prev_end is not None else 0
    print(f"{e.time_range.start - t0:10.1f} gap {gap:8.1f} dur {e.time_range.end - e.time_range.start:9.1f}  {e.name[:70]}")
    prev_end = e.time_range.end
cpu = [e for e in prof.events() if e.device_type.name == "CPU"]
agg = {}
for e in cpu:
    agg.setdefault(e.name, [0, 0.0])
    agg[e.name][0] += 1
    agg[e.name][1] += e.time_range.end - e.time_range.start
for k, (n, tot) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:15]:
    print(f"CPU {k[:60]:60s} n={n} total={tot:.0f}us")
b.close()
