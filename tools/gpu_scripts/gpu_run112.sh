cd $GRAFT_REPO_ROOT
for v in "" e1 e2 e3; do GAR_LIB_VARIANT=$v timeout 300 python tools/gram_time.py 19 31 >> gpurun_out/r112.log 2>&1; done
