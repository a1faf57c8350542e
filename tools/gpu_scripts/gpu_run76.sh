cd $GRAFT_REPO_ROOT
GAR_LIB_VARIANT=ldg timeout 300 python tools/check_gram.py > gpurun_out/r76_check.log 2>&1; tail -3 gpurun_out/r76_check.log
for v in "" ldg "" ldg; do GAR_LIB_VARIANT=$v timeout 300 python tools/gram_time.py 7 15 31 47 >> gpurun_out/r76.log 2>&1; done
