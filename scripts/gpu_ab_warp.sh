#!/bin/bash
# A/B of warp-kernel library variants: C4 frame mode, the warp kernel alone (roofline_warp.ms_per_launch)
OUT=gpurun_out; mkdir -p $OUT
for r in 1 2; do for lib in "$@"; do
  DMSGM_LIB_PATH=$lib timeout 300 python bench.py --motion frame --steps 1000 --warmup 20 --no-e2e --no-cpu-baseline > $OUT/abw.json 2>$OUT/abw.err
  python -c "import json; b=json.loads(open('$OUT/abw.json').read().strip().splitlines()[-1]); print('$lib', 'warp us', round(1000*b['roofline_warp']['ms_per_launch'],1), 'step us', round(1000*b['ms_per_step'],1))" || tail -3 $OUT/abw.err
done; done
