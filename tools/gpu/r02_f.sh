#!/bin/bash
# Round-2 GPU pass F: IL=1 + single-sided clamp; bench lines for every config (device-side drains).
set -x
O=gpurun_out/r02f; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
PARITY_STATS=$O/parity.json timeout 1200 python -m pytest tests -x -q -m gpu --deselect tests/test_gpu_longhorizon.py::test_million_step_drift > $O/pytest_gpu.log 2>&1; echo "pytest_rc=$?" >> $O/pytest_gpu.log
for c in C3 C5 C2 C4; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 600 python bench.py --config C3 --eager --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_C3_eager.json 2> $O/bench_C3_eager.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
ls -la $O
