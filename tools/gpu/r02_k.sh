#!/bin/bash
O=gpurun_out/r02k; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke_rc=$?" >> $O/smoke.log
PARITY_STATS=$O/parity.json timeout 1500 python -m pytest tests -x -q -m gpu --deselect tests/test_gpu_longhorizon.py::test_million_step_drift > $O/pytest_gpu.log 2>&1; echo "pytest_rc=$?" >> $O/pytest_gpu.log
