#!/bin/bash
# Frame-warp (NEXT-3) iteration: warp parity tests, C4 bench in frame mode, one ncu capture of the warp kernel.
TAG=${1:-warp}
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_warp.py -m gpu -q -rf > $OUT/pytest_warp_$TAG.log 2>&1; echo "pytest rc=$?"
tail -3 $OUT/pytest_warp_$TAG.log
timeout 600 python bench.py --motion frame --steps 1000 --warmup 20 --no-e2e --no-cpu-baseline > $OUT/bench_${TAG}_C4mc.json 2> $OUT/bench_${TAG}_C4mc.err; echo "bench rc=$?"
tail -1 $OUT/bench_${TAG}_C4mc.json | cut -c1-300
python -c "import json; b=json.loads(open('$OUT/bench_${TAG}_C4mc.json').read().strip().splitlines()[-1]); print(json.dumps(b.get('roofline_warp'))[:600])"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dmsgm_warp -s 4 -c 1 \
  -o $OUT/prof_$TAG -f python bench.py --motion frame --steps 4 --warmup 5 --no-e2e --no-cpu-baseline \
  > $OUT/ncu_full_$TAG.log 2>&1; echo "ncu rc=$?"
