# Register-blocked CUDA-core Gram (gram_ccb.cuh): accuracy, time per pass against the tensor cores, parity suite, C5 sweep
cd $GRAFT_REPO_ROOT
o=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1 || { tail -20 $o/build.log; exit 1; }
timeout 600 python tools/check_gram.py > $o/check_gram_ccb.log 2>&1; echo "check_gram rc=$?"; cat $o/check_gram_ccb.log | head -20
NS="13 15 16 19 23 24 27 31 32 33 35 37 39 40"
rm -f $o/ccb.log
GAR_GRAM_CC=1 timeout 300 python tools/gram_time.py $NS 2>&1 | tail -1 | tee -a $o/ccb.log
GAR_GRAM_CC=0 timeout 300 python tools/gram_time.py $NS 2>&1 | tail -1 | tee -a $o/ccb.log
GAR_LIB_VARIANT=nopre GAR_GRAM_CC=1 timeout 300 python tools/gram_time.py $NS 2>&1 | tail -1 | tee -a $o/ccb.log
timeout 1500 python -m pytest tests -m gpu -x -q > $o/ccb_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $o/ccb_pytest.log
timeout 600 python tools/sweep.py > $o/ccb_sweep_C5.log 2>&1; echo "sweep rc=$?"; head -24 $o/ccb_sweep_C5.log
