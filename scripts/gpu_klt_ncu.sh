# KLT: tests + timing + one full ncu capture per heavy kernel (LK, score, select) with source
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-klt}
bash scripts/gpu_klt_check.sh $TAG
for k in klt_lk_kernel klt_score_stream_kernel klt_select_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o $OUT/prof_${TAG}_$k -f \
    python scripts/klt_time.py C4ring 1 > $OUT/ncu_${TAG}_$k.log 2>&1; echo "ncu $k rc=$?"
done
