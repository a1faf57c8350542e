cd $GRAFT_REPO_ROOT
timeout 300 python tools/check_gram.py > gpurun_out/r52_check_gram.log 2>&1; echo "rc=$?" >> gpurun_out/r52_check_gram.log
for v in "" exp1 base; do GAR_LIB_VARIANT=$v timeout 300 python tools/gram_time.py 7 15 31 35 63 >> gpurun_out/r52.log 2>&1; done
