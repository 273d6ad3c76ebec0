#!/bin/bash
# Round-2 GPU pass D: bench C3 / C2 with the interleaved kernel, ncu of C3.
set -x
O=gpurun_out/r02d; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_C3.json 2> $O/bench_C3.err
timeout 600 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_C2.json 2> $O/bench_C2.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bocd_update -s 3 -c 1 -o $O/c3 \
  python bench.py --config C3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_c3.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bocd_update -s 300 -c 1 -o $O/c5 \
  python bench.py --config C5 --steps 1 --warmup 1 --calls 400 --no-e2e --no-cpu-baseline > $O/ncu_c5.log 2>&1
ls -la $O
