cd $GRAFT_REPO_ROOT
for v in "" p3 p5; do GAR_LIB_VARIANT=$v timeout 300 python tools/gram_time.py 35 47 63 >> gpurun_out/r54.log 2>&1; done
