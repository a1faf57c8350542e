cd $GRAFT_REPO_ROOT
timeout 300 python tools/check_gram.py > gpurun_out/r38_check_gram.log 2>&1; echo "rc=$?" >> gpurun_out/r38_check_gram.log
timeout 300 python tools/gram_time.py 3 7 11 15 19 31 35 47 63 >> gpurun_out/r38.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "gram or distances or krum or bulyan" > gpurun_out/r38_pytest.log 2>&1; tail -3 gpurun_out/r38_pytest.log
