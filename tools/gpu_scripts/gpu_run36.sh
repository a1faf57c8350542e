cd $GRAFT_REPO_ROOT
timeout 300 python tools/check_gram.py > gpurun_out/r36_check_gram.log 2>&1; echo "rc=$?" >> gpurun_out/r36_check_gram.log
for wl in C3 sweep:7 sweep:15 sweep:47 sweep:63; do timeout 300 python tools/ab_step.py $wl >> gpurun_out/r36_ab.log 2>&1; done
