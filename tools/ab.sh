# A/B timing of alternative builds / kernel variants on one GPU (tuning only).
#   VARIANTS="kg4 kg8:128x8s3 ..." bash tools/ab.sh    (NAME[:FALCON_BOCD_VARIANT][:units])
#   builds from tools/tune_build.py; ":units" sets FALCON_BOCD_GRID_UNITS (one unit per CTA)
mkdir -p gpurun_out
for spec in $VARIANTS; do
  IFS=: read -r v kv gu <<< "$spec"
  for rep in 1 2; do
    if [ -n "$gu" ]; then export FALCON_BOCD_GRID_UNITS=1; else unset FALCON_BOCD_GRID_UNITS; fi
    FALCON_BOCD_VARIANT=$kv FALCON_BOCD_LIB=tune/$v/libfalcon_bocd.so timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline ${BENCH_ARGS:-} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$spec', round(d['ms_per_step'],2), '%.4g' % d['value'], d['clocks']['sm_mhz'])"
  done
done
unset FALCON_BOCD_GRID_UNITS
