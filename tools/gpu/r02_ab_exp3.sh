#!/bin/bash
O=gpurun_out/ab; mkdir -p $O; rm -f $O/ab_C2.txt $O/ab_C3.txt $O/ab_C4.txt
VARIANTS="base exp3" CFG=C3 bash tools/gpu/ab_c3.sh
VARIANTS="base exp3" CFG=C4 bash tools/gpu/ab_c3.sh
VARIANTS="base exp3" CFG=C2 STEPS=5 bash tools/gpu/ab_c3.sh
FALCON_BOCD_LIB=tune/exp3/libfalcon_bocd.so PARITY_STATS=$O/exp3_parity_stats.json LONGHORIZON_OUT=$O/exp3_longhorizon.json timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_longhorizon.py -q -x > $O/exp3_parity.log 2>&1; tail -2 $O/exp3_parity.log
