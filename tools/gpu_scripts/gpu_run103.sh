cd $GRAFT_REPO_ROOT
for v in "" prestage "" prestage; do GAR_LIB_VARIANT=$v timeout 300 python tools/gram_time.py 15 31 47 >> gpurun_out/r103.log 2>&1; done
