#!/bin/bash
# A/B timing of kernel variants selected by env vars (no tests).  Usage: bash scripts/gpu_ab.sh TAG "ENV1" "ENV2" ...
TAG=$1; shift
OUT=gpurun_out; mkdir -p $OUT
for cfg in ${CONFIGS:-C4}; do
for v in "$@"; do
  env $v timeout 300 python bench.py --config $cfg --steps 2000 --warmup 20 --no-e2e --no-cpu-baseline > $OUT/ab_${TAG}.json 2>$OUT/ab_${TAG}.err
  python -c "import json; b=json.loads(open('$OUT/ab_${TAG}.json').read().strip().splitlines()[-1]); print('$cfg', '[$v]', round(b['value']), 'fps', 'us/step', round(1000*b['ms_per_step'],1), 'frac', round(b['roofline']['frac'],3))" || tail -3 $OUT/ab_${TAG}.err
done
done
