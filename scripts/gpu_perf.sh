#!/bin/bash
# Faster iteration pass: gpu tests (quick subset unless FULL=1), bench (no e2e/cpu), one ncu --set full capture.
TAG=${1:-perf}
OUT=gpurun_out
mkdir -p $OUT
if [ "${FULL:-0}" = "1" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -rf > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
else
  timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -x > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
fi
tail -3 $OUT/pytest_gpu_$TAG.log
for cfg in ${CONFIGS:-C4}; do
  timeout 600 python bench.py --config $cfg --steps 2000 --warmup 20 --no-e2e --no-cpu-baseline > $OUT/bench_${TAG}_$cfg.json 2> $OUT/bench_${TAG}_$cfg.err; echo "bench $cfg rc=$?"
  python -c "import json,sys; b=json.loads(open('$OUT/bench_${TAG}_$cfg.json').read().strip().splitlines()[-1]); print('$cfg', round(b['value']), b['unit'], 'ms/step', round(b['ms_per_step'],4), 'GB/s', round(b['roofline']['achieved']), 'frac', round(b['roofline']['frac'],3), 'clk', b['clocks']['sm_mhz'])"
done
if [ "${NCU:-1}" = "1" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dmsgm_step -s 8 -c 1 \
  -o $OUT/prof_$TAG -f python bench.py --steps 4 --warmup 5 --no-e2e --no-cpu-baseline \
  > $OUT/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
fi
