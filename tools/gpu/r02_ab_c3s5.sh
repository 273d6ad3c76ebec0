#!/bin/bash
O=gpurun_out/ab; mkdir -p $O; rm -f $O/ab_C3.txt
VARIANTS="base c3s5" CFG=C3 bash tools/gpu/ab_c3.sh
