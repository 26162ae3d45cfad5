#!/bin/bash
# A/B timing of library variants, interleaved, REPS rounds.  Each argument is LIB[:ENV=VAL[,ENV=VAL]]
# Usage: CONFIGS="C4 C5" REPS=2 bash scripts/gpu_ablib.sh lib1.so lib2.so:DMSGM_STAGED_OCC=4 ...
OUT=gpurun_out; mkdir -p $OUT
for r in $(seq 1 ${REPS:-2}); do
for cfg in ${CONFIGS:-C4}; do
for v in "$@"; do
  lib=${v%%:*}; envs=""; [ "$lib" != "$v" ] && envs=$(echo ${v#*:} | tr ',' ' ')
  steps=2000; [ "$cfg" = "C5" ] && steps=500
  env DMSGM_LIB_PATH=$lib $envs timeout 300 python bench.py --config $cfg --steps $steps --warmup 20 --no-e2e --no-cpu-baseline > $OUT/ablib.json 2>$OUT/ablib.err
  python -c "import json; b=json.loads(open('$OUT/ablib.json').read().strip().splitlines()[-1]); print('$cfg', '$v', 'us/step', round(1000*b['ms_per_step'],2), 'frac', round(b['roofline']['frac'],3), b['clocks']['sm_mhz'])" || tail -3 $OUT/ablib.err
done; done; done
