# tf32 Gram with the n-sized raw ring: accuracy, one pass per n (vs the fixed-depth geometry), parity suite
cd $GRAFT_REPO_ROOT
o=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1 || { tail -20 $o/build.log; exit 1; }

NS="7 11 15 19 23 27 31 35 39 43 47 55 63"
rm -f $o/ring.log
timeout 300 python tools/gram_time.py $NS 2>&1 | tail -1 | tee -a $o/ring.log

timeout 600 python tools/check_gram.py > $o/check_gram.log 2>&1; echo "check_gram rc=$?"; tail -5 $o/check_gram.log
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider > $o/pytest_all.log 2>&1; echo "all pytest rc=$?"; tail -4 $o/pytest_all.log
