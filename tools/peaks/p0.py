"""P0: the FP64 pipe peak with the SM clock sampled by nvidia-smi during the DFMA loop.

    python tools/peaks/p0.py > profiles/r02_p0_fp64_peaks.json

DFMA per clock per SM = dfma_per_s / (SMs x median sampled SM clock while the loop runs).
"""
import json
import os
import subprocess
import sys
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from bench import ClockSampler  # noqa: E402

binp = os.path.join(HERE, "fp64_peak")
if not os.path.exists(binp):
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", binp, binp + ".cu"])
with ClockSampler(0) as clk:
    out = subprocess.run([binp, "60"], capture_output=True, text=True, check=True).stdout
d = json.loads(out.strip().splitlines()[-1])
cs = clk.summary()
d["clocks_during_run"] = cs
if cs.get("sm_mhz"):
    d["dfma_per_clk_per_sm"] = d["dfma_per_s"] / (d["sms"] * cs["sm_mhz"] * 1e6)
    d["nominal_per_s_at_sampled_clock"] = d["sms"] * 64 * cs["sm_mhz"] * 1e6
d["note"] = ("clock = median nvidia-smi sample during the run (includes the transcendental loops); "
             "nominal FP64 = SMs x 64 lanes/clk x clock")
print(json.dumps(d))
