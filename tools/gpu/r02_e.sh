#!/bin/bash
# Round-2 GPU pass E: octet-interleaved kernel; timeline diagnostic of the bench loop.
set -x
O=gpurun_out/r02e; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python tools/diag/trace_steps.py C2 4 > $O/trace_c2.txt 2>&1
timeout 600 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_C3.json 2> $O/bench_C3.err
timeout 600 python bench.py --config C5 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > $O/bench_C5.json 2> $O/bench_C5.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bocd_update -s 3 -c 1 -o $O/c3 \
  python bench.py --config C3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_c3.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > $O/pytest_parity.log 2>&1
ls -la $O
