#!/bin/bash
# Row-band (C5b) GPU pass: band parity tests, 1-GPU band benches, torchrun path on one GPU.
OUT=gpurun_out; mkdir -p $OUT
TAG=${1:-band}
timeout 900 python -m pytest tests/test_gpu_band.py -q -rf -x > $OUT/pytest_$TAG.log 2>&1; echo "band tests rc=$?"
tail -3 $OUT/pytest_$TAG.log
for G in 1 2 4 8; do
  timeout 300 python bench.py --config C5b --bands $G --steps 2000 --warmup 24 --no-cpu-baseline > $OUT/bench_${TAG}_g$G.json 2>&1
  echo "G=$G rc=$?"; tail -1 $OUT/bench_${TAG}_g$G.json | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['ms_per_step']*1e3, 'us/step', j['value'], j['e2e'], j['band_status'])" 2>&1 | tail -2
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --config C5b --dist-backend gloo --same-device --steps 200 --warmup 8 --no-cpu-baseline > $OUT/bench_${TAG}_torchrun2.json 2>&1
echo "torchrun2 rc=$?"; tail -3 $OUT/bench_${TAG}_torchrun2.json | cut -c1-700
