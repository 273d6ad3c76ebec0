#!/bin/bash
O=gpurun_out/ab; mkdir -p $O; rm -f $O/ab_C2.txt $O/ab_C3.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "balanced or persistent_kernels" > $O/wide_parity.log 2>&1; tail -2 $O/wide_parity.log
VARIANTS="base wide" CFG=C2 STEPS=5 bash tools/gpu/ab_c3.sh
VARIANTS="base wide" CFG=C3 bash tools/gpu/ab_c3.sh
