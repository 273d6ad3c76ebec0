#!/bin/bash
O=gpurun_out/ab; mkdir -p $O; rm -f $O/ab_C3.txt $O/ab_C4.txt
VARIANTS="base keyw0" CFG=C4 BENCH_ARGS=--eager STEPS=2 bash tools/gpu/ab_c3.sh
VARIANTS="base keyw0" CFG=C3 BENCH_ARGS=--eager bash tools/gpu/ab_c3.sh
FALCON_BOCD_LIB=tune/keyw0/libfalcon_bocd.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > $O/keyw0_parity.log 2>&1; tail -2 $O/keyw0_parity.log
