"""Builds libfalcon_bocd.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

    python -m paper_2410_12588_b200.build [--force]
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libfalcon_bocd.so")
SOURCES = ["capi.cu", "bocd_kernels.cu", "tracegen.cu", "verify.cu", "groups.cu", "acf.cu"]
HEADERS = ["bocd_kernel.cuh", "bocd_variants.h", "fastmath.cuh", "cellmath.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-O2", f"-I{os.path.join(ROOT, 'include')}"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps += [os.path.join(ROOT, "include", f) for f in ("falcon_bocd.h", "falcon_trace.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, lib: str = LIB, defines: tuple = (), extra: tuple = ()) -> str:
    """Builds the library; `lib`/`defines` give alternative builds for A/B tuning (tools/tune_build.py)."""
    if not force and lib == LIB and not _stale():
        return LIB
    objdir = os.path.join(os.path.dirname(lib), "build") if lib != LIB else os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [NVCC, *FLAGS, *extra, *[f"-D{d}" for d in defines], "-Xptxas", "-v", "-c", os.path.join(CSRC, src), "-o", obj]
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{p.stderr}")
        with open(obj + ".ptxas.txt", "w") as f:
            f.write(p.stderr)
        if verbose:
            sys.stderr.write(p.stderr)
        return obj

    with ThreadPoolExecutor(len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = lib + ".tmp"
    subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs])
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
