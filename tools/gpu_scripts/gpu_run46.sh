cd $GRAFT_REPO_ROOT
for v in "" c16 c16e1 base; do GAR_LIB_VARIANT=$v timeout 300 python tools/gram_time.py 7 31 63 >> gpurun_out/r46.log 2>&1; done
