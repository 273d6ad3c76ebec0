#!/bin/bash
O=gpurun_out/ab; mkdir -p $O; rm -f $O/ab_C2.txt
VARIANTS="base kg4" CFG=C2 STEPS=5 bash tools/gpu/ab_c3.sh
