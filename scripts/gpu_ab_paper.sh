# A/B of the per-pixel path (N = 1): the paper pipeline (C4p + Gaussian/median + frame warp) and plain C4p, default lib vs a BPT-2 build (ablib_n1b2.so)
OUT=gpurun_out
for r in 1 2; do for lib in paper_1702_05156_b200/libdmsgm.so ./ablib_n1b2.so; do
  DMSGM_LIB_PATH=$lib timeout 300 python bench.py --config C4p --prefilter 5,1.0,1 --motion frame --steps 1000 --warmup 20 --no-e2e --no-cpu-baseline > $OUT/abp.json 2>$OUT/abp.err
  python -c "import json; b=json.loads(open('$OUT/abp.json').read().strip().splitlines()[-1]); print('$lib paper', round(1000*b['ms_per_step'],1))"
  DMSGM_LIB_PATH=$lib timeout 300 python bench.py --config C4p --steps 1000 --warmup 20 --no-e2e --no-cpu-baseline > $OUT/abp.json 2>$OUT/abp.err
  python -c "import json; b=json.loads(open('$OUT/abp.json').read().strip().splitlines()[-1]); print('$lib C4p', round(1000*b['ms_per_step'],1))"
done; done
