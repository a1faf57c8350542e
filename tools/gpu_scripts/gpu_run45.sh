cd $GRAFT_REPO_ROOT
for v in "" exp1 exp6 exp7 exp8; do GAR_LIB_VARIANT=$v timeout 300 python tools/gram_time.py 7 31 63 >> gpurun_out/r45.log 2>&1; done
