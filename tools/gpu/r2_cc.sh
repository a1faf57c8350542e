# CUDA-core Gram (gram_cc.cu): accuracy, time per pass against the tensor-core kernel; parity suite
cd $GRAFT_REPO_ROOT
o=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1 || { tail -20 $o/build.log; exit 1; }
timeout 600 python tools/check_gram.py > $o/check_gram_cc.log 2>&1; echo "check_gram rc=$?"; head -14 $o/check_gram_cc.log
NS="3 5 7 8 9 10 11 12 13 16"
rm -f $o/cc.log
timeout 300 python tools/gram_time.py $NS 2>&1 | tail -1 | tee -a $o/cc.log
GAR_GRAM_CC=0 timeout 300 python tools/gram_time.py $NS 2>&1 | tail -1 | tee -a $o/cc.log
timeout 1500 python -m pytest tests -m gpu -x -q > $o/cc_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $o/cc_pytest.log
timeout 600 python tools/sweep.py > $o/cc_sweep_C5.log 2>&1; echo "sweep rc=$?"; tail -30 $o/cc_sweep_C5.log
