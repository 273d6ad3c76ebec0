#!/bin/bash
# ncu capture of the C2 update kernel only (the balanced one-CTA-per-SM launch), CSV export.
O=gpurun_out/r02ncu; mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bocd_update -s 3 -c 1 -o /tmp/c2 \
  python bench.py --config C2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_c2.log 2>&1
ncu -i /tmp/c2.ncu-rep --page raw --csv > $O/c2.raw.csv 2>/dev/null
ncu -i /tmp/c2.ncu-rep --page source --csv --print-source sass > $O/c2.src.csv 2>/dev/null
gzip -f $O/c2.src.csv
