cd $GRAFT_REPO_ROOT
for v in exp10 exp11 exp8 exp1; do GAR_LIB_VARIANT=$v timeout 300 python tools/gram_time.py 7 31 63 >> gpurun_out/r53.log 2>&1; done
