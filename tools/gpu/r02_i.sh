#!/bin/bash
O=gpurun_out/r02i; mkdir -p $O
VARIANTS="cur znorm" bash tools/gpu/ab_c3.sh > $O/ab.txt 2>&1
FALCON_BOCD_LIB=tune/znorm/libfalcon_bocd.so timeout 900 ncu --set full --import-source on --clock-control none -k regex:bocd_update -s 3 -c 1 -o $O/c3 \
  python bench.py --config C3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_c3.log 2>&1
FALCON_BOCD_LIB=tune/znorm/libfalcon_bocd.so timeout 900 ncu --set full --import-source on --clock-control none -k regex:bocd_update -s 3 -c 1 -o $O/c4 \
  python bench.py --config C4 --series 12500 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_c4.log 2>&1
