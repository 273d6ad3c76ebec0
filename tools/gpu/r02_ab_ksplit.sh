#!/bin/bash
O=gpurun_out/ab; mkdir -p $O; rm -f $O/ab_C3.txt $O/ab_C4.txt
VARIANTS="base ksplit" CFG=C3 bash tools/gpu/ab_c3.sh
VARIANTS="base ksplit" CFG=C4 bash tools/gpu/ab_c3.sh
FALCON_BOCD_LIB=tune/ksplit/libfalcon_bocd.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x > $O/ksplit_parity.log 2>&1; tail -2 $O/ksplit_parity.log
