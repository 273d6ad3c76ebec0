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
# ncu: one steady-state launch of each update kernel (full set with source); then the launch list
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bocd_update -s 3 -c 1 -o $O/c3 \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_c3.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bocd_update -s 3 -c 1 -o $O/c4 \
  python bench.py --config C4 --series 12500 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_c4.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bocd_update -s 3 -c 1 -o $O/c2 \
  python bench.py --config C2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_c2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bocd_update -s 2500 -c 1 -o $O/c5 \
  python bench.py --config C5 --steps 1 --warmup 2 --no-e2e --no-cpu-baseline > $O/ncu_c5.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launches.log 2>&1
ls -la $O
