#!/bin/bash
O=gpurun_out/ab; mkdir -p $O; rm -f $O/ab_C2.txt $O/ab_C3.txt $O/ab_C4.txt $O/ab_C5.txt
VARIANTS="base log2" CFG=C3 bash tools/gpu/ab_c3.sh
VARIANTS="base log2" CFG=C4 bash tools/gpu/ab_c3.sh
VARIANTS="base log2" CFG=C2 STEPS=5 bash tools/gpu/ab_c3.sh
VARIANTS="base log2" CFG=C5 STEPS=3 bash tools/gpu/ab_c3.sh
for v in base log2; do
FALCON_BOCD_LIB=tune/$v/libfalcon_bocd.so PARITY_STATS=$O/${v}_parity_stats.json LONGHORIZON_OUT=$O/${v}_longhorizon.json timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_longhorizon.py tests/test_gpu_fastmath.py -q -x > $O/${v}_parity.log 2>&1; tail -2 $O/${v}_parity.log
done
