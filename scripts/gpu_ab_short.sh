#!/bin/bash
# A/B of library variants on short timed regions (K = 200 steps: the full-clock plateau, before the
# board's power cap), interleaved, REPS rounds; prints value and replay median (us/step).
# Usage: CONFIGS="C4 C4p" REPS=3 bash scripts/gpu_ab_short.sh lib1.so lib2.so[:ENV=VAL,...] ...
OUT=gpurun_out; mkdir -p $OUT
for r in $(seq 1 ${REPS:-3}); do
for cfg in ${CONFIGS:-C4}; do
for v in "$@"; do
  lib=${v%%:*}; envs=""; [ "$lib" != "$v" ] && envs=$(echo ${v#*:} | tr ',' ' ')
  env DMSGM_LIB_PATH=$lib $envs timeout 300 python bench.py --config $cfg --steps 200 --warmup 20 --no-e2e --no-cpu-baseline > $OUT/abs.json 2>$OUT/abs.err
  python -c "import json; b=json.loads(open('$OUT/abs.json').read().strip().splitlines()[-1]); print('$cfg', '$v', 'us/step', round(1000*b['ms_per_step'],2), 'median', round(1000*b['median_ms_per_step'],2), b['clocks']['sm_mhz'])" || tail -3 $OUT/abs.err
done; done; done
