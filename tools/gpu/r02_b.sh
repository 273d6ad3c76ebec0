#!/bin/bash
# Round-2 GPU pass B: shared-memory probe, P0 FP64 peak with sampled clocks, C5 and EAGER bench
# lines, the million-step precision test.
set -x
O=gpurun_out/r02b; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python tools/peaks/p0.py > $O/p0.json 2> $O/p0.err
timeout 600 python bench.py --config C5 --steps 5 --warmup 3 > $O/bench_C5.json 2> $O/bench_C5.err
timeout 600 python bench.py --config C3 --eager --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_C3_eager.json 2> $O/bench_C3_eager.err
timeout 600 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_C3.json 2> $O/bench_C3.err
LONGHORIZON_OUT=$O/longhorizon.json PARITY_STATS=$O/parity_long.json timeout 1500 python -m pytest tests/test_gpu_longhorizon.py -x -q > $O/longhorizon.log 2>&1
ls -la $O
