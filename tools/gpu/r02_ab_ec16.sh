#!/bin/bash
O=gpurun_out/ab; mkdir -p $O; rm -f $O/ab_C4.txt
VARIANTS="base ec16" CFG=C4 bash tools/gpu/ab_c3.sh
FALCON_BOCD_LIB=tune/ec16/libfalcon_bocd.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "large_R or persistent or priors" > $O/ec16_parity.log 2>&1; tail -2 $O/ec16_parity.log
