#!/bin/bash
# Round-2 GPU pass G: integer-alpha / half-log FULL kernels: GPU tests + A/B vs the previous build.
O=gpurun_out/r02g; mkdir -p $O
PARITY_STATS=$O/parity.json timeout 1200 python -m pytest tests -x -q -m gpu --deselect tests/test_gpu_longhorizon.py::test_million_step_drift > $O/pytest_gpu.log 2>&1; echo "pytest_rc=$?" >> $O/pytest_gpu.log
VARIANTS="clamp1 ai" bash tools/gpu/ab_c3.sh > $O/ab.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bocd_update -s 3 -c 1 -o $O/c3 \
  python bench.py --config C3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_c3.log 2>&1
