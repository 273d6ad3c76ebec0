# A/B timing of alternative builds on one GPU (tuning only).
#   VARIANTS="base exp1 ..." bash tools/ab.sh    (NAME = a build from tools/tune_build.py)
mkdir -p gpurun_out
for v in $VARIANTS; do
  for rep in 1 2; do
    FALCON_BOCD_LIB=tune/$v/libfalcon_bocd.so timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline ${BENCH_ARGS:-} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$v', round(d['ms_per_step'],2), '%.4g' % d['value'], d['clocks']['sm_mhz'])"
  done
done
