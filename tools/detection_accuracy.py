"""Detection accuracy of the GPU detectors on labelled synthetic traces (
PAPER.md Tables 5-6 define the scores).  One GPU:

    python tools/detection_accuracy.py [S] [T] [config]   -> one JSON line (profiles/)

Detectors, per series (a link or a rank; ground truth = the generator's injected episodes):
  raw BOCD : any PROB change point (p_new > 0.9) at t >= 1;
  BOCD+V   : any verified DEGRADE change point paired into a fail-slow event (the 10%
             before/after rule of P:772-779 + pairing, readings V1-V5).
Change points are PROB events (p_new > 0.9), or PROB + MAP resets.  delay_steps: from the
first injected onset to the first flag (raw: the event's step; BOCD+V: the step at which the
verification's after-window is complete), over series flagged at or after their onset.
SlideWindow (the paper's comparison baseline) is out of scope.
"""
import json
import os
import sys


sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_12588_b200 import detection, tracegen  # noqa: E402


def main():
    S = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
    T = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
    name = sys.argv[3] if len(sys.argv) > 3 else "C3"
    sigma = float(sys.argv[4]) if len(sys.argv) > 4 else None
    cfg = tracegen.CONFIGS[name]
    spec = tracegen.make_spec(cfg, n_series=S, T=T, sigma=sigma)
    out = detection.evaluate(spec, cfg, T)
    out["note"] = ("synthetic labelled traces (tracegen); detectors: raw BOCD change points (PROB = "
                   "p_new > 0.9, optionally + MAP resets) and the same verified by the 10% rule and "
                   "paired (BOCD+V); the paper's Tables 5-6 are context only")
    print(json.dumps(out))


if __name__ == "__main__":
    main()
