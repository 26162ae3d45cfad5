#!/bin/bash
# A/B of prefilter library variants: C4 + prefilter, the filter kernel alone (roofline.ms_per_launch)
OUT=gpurun_out; mkdir -p $OUT
for r in 1 2; do for lib in "$@"; do
  DMSGM_LIB_PATH=$lib timeout 300 python bench.py --prefilter 5,1.0,1 --steps 1000 --warmup 20 --no-e2e --no-cpu-baseline > $OUT/abpf.json 2>$OUT/abpf.err
  python -c "import json; b=json.loads(open('$OUT/abpf.json').read().strip().splitlines()[-1]); print('$lib', 'filter us', round(1000*b['roofline']['ms_per_launch'],1), 'step us', round(1000*b['ms_per_step'],1))" || tail -3 $OUT/abpf.err
done; done
