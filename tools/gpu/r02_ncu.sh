#!/bin/bash
# ncu captures of the update kernels, exported on the box to CSV (raw metrics + SASS source
# page) so that only text comes back (gpurun copies back <= 64 MiB); then the launch list.
O=gpurun_out/r02ncu; mkdir -p $O
cap() {  # name, ncu launch-skip, bench args...
  local n=$1 skip=$2; shift 2
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:bocd_update -s $skip -c 1 -o /tmp/$n \
    python bench.py "$@" --no-e2e --no-cpu-baseline > $O/ncu_$n.log 2>&1
  ncu -i /tmp/$n.ncu-rep --page raw --csv > $O/$n.raw.csv 2>/dev/null
  ncu -i /tmp/$n.ncu-rep --page source --csv --print-source sass > $O/$n.src.csv 2>/dev/null
  rm -f /tmp/$n.ncu-rep
}
cap c3 3 --steps 1 --warmup 3
cap c4 3 --config C4 --series 12500 --steps 1 --warmup 3
cap c2 3 --config C2 --steps 1 --warmup 3
cap c5 2500 --config C5 --steps 1 --warmup 2
cap c3e 3 --eager --steps 1 --warmup 3
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launches.log 2>&1
gzip -f $O/*.src.csv
ls -la $O
