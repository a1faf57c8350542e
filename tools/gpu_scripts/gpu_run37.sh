cd $GRAFT_REPO_ROOT
for v in "" exp1 exp2 exp3 exp4; do GAR_LIB_VARIANT=$v timeout 300 python tools/gram_time.py 7 15 31 35 47 63 >> gpurun_out/r37.log 2>&1; done
