#!/bin/bash
O=gpurun_out/ab; mkdir -p $O; rm -f $O/ab_C2.txt
VARIANTS="base c2j4" CFG=C2 STEPS=5 bash tools/gpu/ab_c3.sh
FALCON_BOCD_LIB=tune/c2j4/libfalcon_bocd.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "c2 or balanced or persistent or permutation" > $O/c2j4_parity.log 2>&1; tail -2 $O/c2j4_parity.log
