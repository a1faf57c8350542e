cd $GRAFT_REPO_ROOT
for v in base "" fixed u2 u3fixed base; do GAR_LIB_VARIANT=$v timeout 300 python tools/gram_time.py 7 15 31 35 63 >> gpurun_out/r39b.log 2>&1; done
