# prefilter iteration: parity tests, the filter A/B line, one full ncu capture of the filter
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-pf}
timeout 600 python -m pytest tests/test_gpu_prefilter.py tests/test_gpu_pdl.py -q -x > $OUT/pf_tests_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pf_tests_$TAG.log
shift; bash scripts/gpu_ab_pf.sh paper_1702_05156_b200/libdmsgm.so "$@"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dmsgm_prefilter -s 3 -c 1 -o $OUT/prof_$TAG -f python bench.py --prefilter 5,1.0,1 --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_$TAG.log 2>&1; echo "ncu rc=$?"
