# frame-warp iteration: parity tests, the warp A/B line, one full ncu capture of the warp kernel
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-warp}
timeout 900 python -m pytest tests/test_gpu_warp.py tests/test_gpu_pdl.py -q -x > $OUT/warp_tests_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/warp_tests_$TAG.log
shift; bash scripts/gpu_ab_warp.sh paper_1702_05156_b200/libdmsgm.so "$@"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dmsgm_warp -s 4 -c 1 -o $OUT/prof_$TAG -f python bench.py --motion frame --steps 4 --warmup 5 --no-e2e --no-cpu-baseline > $OUT/ncu_$TAG.log 2>&1; echo "ncu rc=$?"
