cd $GRAFT_REPO_ROOT
timeout 300 python tools/check_gram.py > gpurun_out/r111_check.log 2>&1; echo "rc=$?" >> gpurun_out/r111_check.log; cat gpurun_out/r111_check.log
for v in 1 0 1 0; do GAR_GRAM_I8=$v timeout 300 python tools/gram_time.py 19 23 27 31 >> gpurun_out/r111.log 2>&1; done
