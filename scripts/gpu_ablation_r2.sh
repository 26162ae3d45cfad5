# round-2 SURVEY §8(d) ablation: parity of the ablation builds, then every variant timed + one ncu launch
OUT=gpurun_out; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x > $OUT/abl_parity_default.log 2>&1; echo "parity(default build, all kernel paths) rc=$?"; tail -1 $OUT/abl_parity_default.log
for lib in abl/lib_scalar.so abl/lib_evict.so abl/lib_notilde.so abl/lib_nofinish.so; do
  DMSGM_LIB_PATH=$lib timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "default" > $OUT/abl_parity.log 2>&1; echo "parity $lib rc=$?"; tail -1 $OUT/abl_parity.log
done
bash scripts/gpu_ablation.sh paper_1702_05156_b200/libdmsgm.so \
  paper_1702_05156_b200/libdmsgm.so:DMSGM_KERNEL=generic,DMSGM_GENERIC_BPT=1 \
  paper_1702_05156_b200/libdmsgm.so:DMSGM_KERNEL=generic,DMSGM_GENERIC_BPT=2 \
  paper_1702_05156_b200/libdmsgm.so:DMSGM_KERNEL=generic,DMSGM_GENERIC_BPT=4 \
  abl/lib_scalar.so abl/lib_evict.so abl/lib_notilde.so abl/lib_nofinish.so \
  paper_1702_05156_b200/libdmsgm.so:DMSGM_PDL=0
