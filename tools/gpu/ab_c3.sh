#!/bin/bash
# A/B timing of tune/ builds on the C3 bench (kernel ms per 1,000-step call).  VARIANTS env.
O=gpurun_out/ab; mkdir -p $O
for rep in 1 2; do
  for v in $VARIANTS; do
    FALCON_BOCD_LIB=tune/$v/libfalcon_bocd.so timeout 300 python bench.py --config ${CFG:-C3} --steps ${STEPS:-3} --warmup 2 --no-e2e --no-cpu-baseline ${BENCH_ARGS:-} 2> $O/$v.err | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$v', round(d['roofline']['kernel_ms_avg'],3), round(d['ms_per_step'],3), '%.4g' % d['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> $O/ab_${CFG:-C3}.txt 2>&1
  done
done
cat $O/ab_${CFG:-C3}.txt
