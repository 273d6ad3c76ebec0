#!/bin/bash
O=gpurun_out/ab; mkdir -p $O; rm -f $O/ab_C2.txt $O/ab_C3.txt $O/ab_C4.txt
VARIANTS="base ownw" CFG=C3 bash tools/gpu/ab_c3.sh
VARIANTS="base ownw" CFG=C4 bash tools/gpu/ab_c3.sh
FALCON_BOCD_LIB=tune/ownw/libfalcon_bocd.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > $O/ownw_parity.log 2>&1; tail -2 $O/ownw_parity.log
