for cap in 3 2; do for lib in paper_1702_05156_b200/libdmsgm.so ab/libpf_c4m3.so ab/libpf_c4m4.so; do
DMSGM_STAGED_CTAS_PER_SM=$cap DMSGM_LIB_PATH=$lib timeout 300 python scripts/pf_overlap.py 2>&1 | tail -1
done; done
