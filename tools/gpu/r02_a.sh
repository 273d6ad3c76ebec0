#!/bin/bash
# Round-2 GPU pass A: GPU tests, bench lines for every config, ncu captures of the update kernels.
set -x
mkdir -p gpurun_out/r02a
O=gpurun_out/r02a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest_rc=$?" >> $O/pytest_gpu.log
for c in C3 C2 C4 C5; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 600 python bench.py --config C3 --eager --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_C3_eager.json 2> $O/bench_C3_eager.err
# ncu: one steady-state launch of each update kernel (full set, source)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bocd_update -s 3 -c 1 -o $O/c3 \
  python bench.py --config C3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_c3.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bocd_update -s 3 -c 1 -o $O/c4 \
  python bench.py --config C4 --series 12500 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_c4.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bocd_update -s 3 -c 1 -o $O/c2 \
  python bench.py --config C2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_c2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv \
  python bench.py --config C3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1
ls -la $O
