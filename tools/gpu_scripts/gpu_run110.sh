cd $GRAFT_REPO_ROOT
for v in "" v1 v2 v3 ""; do GAR_LIB_VARIANT=$v timeout 300 python tools/gram_time.py 19 31 >> gpurun_out/r110.log 2>&1; done
