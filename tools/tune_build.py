"""Builds alternative copies of libfalcon_bocd.so with extra -D defines for A/B timing runs.

    python tools/tune_build.py NAME DEFINE [DEFINE ...]   ->  tune/NAME/libfalcon_bocd.so
Load one with FALCON_BOCD_LIB=tune/NAME/libfalcon_bocd.so (bench.py / tests).  tune/ is
git-ignored scratch; the product library is always the in-package build.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2410_12588_b200 import build as B  # noqa: E402

if __name__ == "__main__":
    name = sys.argv[1]
    defines = tuple(a for a in sys.argv[2:] if not a.startswith("-"))
    extra = tuple(a for a in sys.argv[2:] if a.startswith("-"))  # raw nvcc flags, e.g. -Xptxas=...
    d = os.path.join(ROOT, "tune", name)
    os.makedirs(d, exist_ok=True)
    print(B.build(force=True, lib=os.path.join(d, "libfalcon_bocd.so"), defines=defines, extra=extra))
