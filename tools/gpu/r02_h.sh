#!/bin/bash
# Round-2 GPU pass H: new parity tests (persistent kernels, priors, thresholds, N3), bench C3.
O=gpurun_out/r02h; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
PARITY_STATS=$O/parity.json timeout 1500 python -m pytest tests -q -m gpu --deselect tests/test_gpu_longhorizon.py::test_million_step_drift > $O/pytest_gpu.log 2>&1; echo "pytest_rc=$?" >> $O/pytest_gpu.log
timeout 600 python -c "
import json
from paper_2410_12588_b200 import detection, tracegen
for name, S, T, sig in (('C3', 512, 6000, 0.05), ('C3', 512, 6000, 0.1), ('C2', 256, 6000, None)):
    cfg = tracegen.CONFIGS[name]
    out = detection.evaluate(tracegen.make_spec(cfg, n_series=S, T=T, sigma=sig), cfg, T)
    print(json.dumps(out))
" > $O/detection.jsonl 2>&1
timeout 600 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_C3.json 2> $O/bench_C3.err
