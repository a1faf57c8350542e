cd $GRAFT_REPO_ROOT
for v in "" exp1 exp2 exp3 exp4; do GAR_LIB_VARIANT=$v timeout 300 python tools/gram_time.py 7 11 15 >> gpurun_out/r94.log 2>&1; done
