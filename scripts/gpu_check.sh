#!/bin/bash
# One GPU pass: smoke, gpu tests, a short bench, ncu launch list (timed region) and one full capture.
# Usage (from the repo root, under gpurun):  bash scripts/gpu_check.sh [tag] [pytest-args...]
TAG=${1:-r01}
shift
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/nvsmi_$TAG.txt 2>&1
lscpu > $OUT/lscpu_$TAG.txt 2>&1
python __graft_entry__.py --smoke > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
timeout 2400 python -m pytest tests -m gpu -q -rf "$@" > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
tail -8 $OUT/pytest_gpu_$TAG.log
timeout 600 python bench.py --steps 2000 --warmup 20 > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"
tail -c 400 $OUT/bench_$TAG.json
timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches_$TAG.csv python bench.py --steps 40 --warmup 5 --no-e2e --no-cpu-baseline \
  > $OUT/ncu_launch_$TAG.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:dmsgm_step -s 8 -c 2 \
  -o $OUT/prof_$TAG -f python bench.py --steps 40 --warmup 5 --no-e2e --no-cpu-baseline \
  > $OUT/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
