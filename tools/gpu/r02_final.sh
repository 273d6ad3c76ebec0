#!/bin/bash
# Round-2 final single-GPU pass: smoke, every GPU test, bench lines, reference arm, ncu captures.
O=gpurun_out/r02final; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke_rc=$?" >> $O/smoke.log
PARITY_STATS=$O/parity_stats.json LONGHORIZON_OUT=$O/longhorizon.json timeout 2400 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest_rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_C3.json 2> $O/bench_C3.err
for c in C2 C4 C5; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 900 python bench.py --eager --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_C3_eager.json 2> $O/bench_C3_eager.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
ls -la $O
