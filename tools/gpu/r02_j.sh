#!/bin/bash
# Round-2 GPU pass J: the software-pipelined FULL kernels: GPU tests + A/B vs the previous build.
O=gpurun_out/r02j; mkdir -p $O
PARITY_STATS=$O/parity.json timeout 1500 python -m pytest tests -x -q -m gpu --deselect tests/test_gpu_longhorizon.py::test_million_step_drift > $O/pytest_gpu.log 2>&1; echo "pytest_rc=$?" >> $O/pytest_gpu.log
rm -f gpurun_out/ab/ab_C3.txt gpurun_out/ab/ab_C4.txt
VARIANTS="cur pipe" bash tools/gpu/ab_c3.sh > $O/ab_c3.txt 2>&1
CFG=C4 STEPS=2 BENCH_ARGS="--series 12500" VARIANTS="cur pipe" bash tools/gpu/ab_c3.sh > $O/ab_c4.txt 2>&1
