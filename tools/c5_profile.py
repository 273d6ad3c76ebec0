"""C5 streaming for an ncu capture of the persistent kernel (one observation per call):

    ncu --set full -k regex:bocd_update -s 12 -c 1 python tools/c5_profile.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_12588_b200 import bocd, tracegen  # noqa: E402

cfg = tracegen.CONFIGS["C5"]
S, calls = 10240, 16
spec = tracegen.make_spec(cfg, n_series=S)
x = torch.empty((S, calls + 1), dtype=torch.float64, device="cuda")
bocd.DeviceTrace(spec, "cuda").generate(x, 0, 0)
b = bocd.BocdBatch(S, R=cfg.R, hazard=cfg.hazard, prior_first_obs=True, prior_cov=cfg.prior_cov)
for t in range(calls):
    b.update_chunk(x[:, t:t + 1].contiguous())
torch.cuda.synchronize()
b.close()
print("ok")
