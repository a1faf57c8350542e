cd $GRAFT_REPO_ROOT
for v in "" spin ops3 ops3spin ""; do GAR_LIB_VARIANT=$v timeout 300 python tools/gram_time.py 7 11 15 31 47 >> gpurun_out/r95.log 2>&1; done
