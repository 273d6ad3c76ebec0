#!/bin/bash
# compute-sanitizer passes (T7) over the small GPU parity cases.  One tool per gpurun call
# (B200_PROFILING.md); usage: tools/sanitize.sh memcheck|racecheck|synccheck|initcheck
set -e
TOOL=${1:-memcheck}
cd "$(dirname "$0")/.."
timeout 1200 compute-sanitizer --tool "$TOOL" --error-exitcode 99 \
  python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "c1_parity or bruteforce or generic_R or chunk_split or nonfinite" \
  > gpurun_out/sanitize_$TOOL.log 2>&1
echo "sanitize $TOOL rc=$?"
