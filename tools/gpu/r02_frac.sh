#!/bin/bash
O=gpurun_out/frac; mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_parity.py -q -x > $O/parity.log 2>&1; tail -2 $O/parity.log
python tools/bench_variants.py > $O/variants.jsonl 2> $O/variants.err
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/c3.json 2> $O/c3.err
