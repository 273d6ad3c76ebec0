#!/bin/bash
O=gpurun_out/ab; mkdir -p $O; rm -f $O/ab_C2.txt $O/ab_C3.txt $O/ab_C4.txt
VARIANTS="fuse fuse2" CFG=C3 bash tools/gpu/ab_c3.sh
VARIANTS="fuse fuse2" CFG=C4 bash tools/gpu/ab_c3.sh
FALCON_BOCD_LIB=tune/fuse2/libfalcon_bocd.so PARITY_STATS=$O/fuse2_parity_stats.json timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x > $O/fuse2_parity.log 2>&1; tail -2 $O/fuse2_parity.log
