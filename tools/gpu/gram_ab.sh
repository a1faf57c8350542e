# Gram A/B: product kernel vs round-1 tf32 kernel (accuracy + time per pass), then gpu tests.
cd $GRAFT_REPO_ROOT
o=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1 || { tail -20 $o/build.log; exit 1; }
bash tools/gram_exp.sh r1 tools/experiments/gram_tc_tf32_r1.cu > $o/gram_exp.log 2>&1 || { tail $o/gram_exp.log; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mmabench tools/mmabench.cu && /tmp/mmabench > $o/mmabench.log 2>&1
timeout 600 python tools/check_gram.py > $o/check_gram.log 2>&1; echo "check_gram rc=$?"; cat $o/check_gram.log
timeout 600 python tools/gram_time.py 7 11 15 19 23 31 35 47 63 2>&1 | tail -1
GAR_LIB_VARIANT=r1 timeout 600 python tools/gram_time.py 7 11 15 19 23 31 35 47 63 2>&1 | tail -1
cat $o/mmabench.log
timeout 1200 python -m pytest tests -q -m gpu -x -p no:cacheprovider > $o/pytest_gram.log 2>&1; echo "pytest rc=$?"; tail -5 $o/pytest_gram.log
