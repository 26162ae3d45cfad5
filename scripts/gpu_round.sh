#!/bin/bash
# Round-end evidence: the standard check (smoke, pytest -m gpu, C4 bench, launch list, ncu)
# plus the other workloads' bench lines.  Usage: bash scripts/gpu_round.sh TAG
TAG=${1:-r33}
OUT=gpurun_out; mkdir -p $OUT
bash scripts/gpu_check.sh $TAG
timeout 600 python bench.py --config C5 --steps 500 --warmup 20 > $OUT/bench_${TAG}_C5.json 2>&1; echo "C5 rc=$?"
timeout 600 python bench.py --config C4p --steps 500 --warmup 20 > $OUT/bench_${TAG}_C4p.json 2>&1; echo "C4p rc=$?"
timeout 600 python bench.py --prefilter 5,1.0,1 --steps 1000 --warmup 20 > $OUT/bench_${TAG}_C4pf.json 2>&1; echo "C4pf rc=$?"
timeout 600 python bench.py --motion frame --steps 1000 --warmup 20 > $OUT/bench_${TAG}_C4mc.json 2>&1; echo "C4mc rc=$?"
timeout 600 python bench.py --motion estimate --steps 200 --warmup 5 > $OUT/bench_${TAG}_C4klt.json 2>&1; echo "C4klt rc=$?"
timeout 600 python bench.py --config C4p --prefilter 5,1.0,1 --motion frame --steps 1000 --warmup 20 > $OUT/bench_${TAG}_paper.json 2>&1; echo "paper rc=$?"
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/bench_${TAG}_C4_K20.json 2>&1; echo "C4 K=20 rc=$?"
for G in 1 8; do timeout 300 python bench.py --config C5b --bands $G --steps 2000 --warmup 24 > $OUT/bench_${TAG}_C5b_g$G.json 2>&1; echo "C5b G=$G rc=$?"; done
# all 64 C5 streams (one launch = the whole C5 batch): scripts/ncu_summary.py TAGc5 --workload C5
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dmsgm_step -s 8 -c 1 \
  -o $OUT/prof_${TAG}c5 -f python bench.py --config C5 --steps 6 --warmup 5 --no-e2e --no-cpu-baseline \
  > $OUT/ncu_full_${TAG}c5.log 2>&1; echo "ncu C5 rc=$?"
for f in C5 C4p C4pf C4mc C4klt paper C4_K20 C5b_g1 C5b_g8; do tail -1 $OUT/bench_${TAG}_$f.json | cut -c1-160; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dmsgm_prefilter -s 3 -c 1 \
  -o $OUT/prof_${TAG}pf -f python bench.py --prefilter 5,1.0,1 --steps 4 --warmup 3 --no-e2e --no-cpu-baseline \
  > $OUT/ncu_full_${TAG}pf.log 2>&1; echo "ncu prefilter rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dmsgm_warp -s 4 -c 1 \
  -o $OUT/prof_${TAG}warp -f python bench.py --motion frame --steps 4 --warmup 5 --no-e2e --no-cpu-baseline \
  > $OUT/ncu_full_${TAG}warp.log 2>&1; echo "ncu warp rc=$?"
