cd $GRAFT_REPO_ROOT
timeout 300 python tools/check_gram.py > gpurun_out/r44_check_gram.log 2>&1; echo "rc=$?" >> gpurun_out/r44_check_gram.log
for v in base "" exp1; do GAR_LIB_VARIANT=$v timeout 300 python tools/gram_time.py 3 7 15 19 31 35 47 63 >> gpurun_out/r44.log 2>&1; done
timeout 300 python tools/gram_prof.py 7 31 63 >> gpurun_out/r44.log 2>&1
