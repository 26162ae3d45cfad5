# KLT iteration: parity tests, timing of the estimate (new build vs the given variants), launch list
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-klt}
timeout 900 python -m pytest tests/test_gpu_klt.py tests/test_gpu_klt_seq.py -q -x -s > $OUT/klt_tests_$TAG.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|Error|assert" $OUT/klt_tests_$TAG.log | tail -5
shift
for lib in paper_1702_05156_b200/libdmsgm.so "$@"; do DMSGM_LIB_PATH=$lib timeout 300 python scripts/klt_time.py C4ring 10 2>&1 | tail -1 | sed "s|^|$lib |"; done
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum --clock-control none --csv -k regex:klt --log-file $OUT/klt_launches_$TAG.csv python scripts/klt_time.py C4ring 1 > /dev/null 2>&1; echo "ncu rc=$?"
