# multi-GPU check: the torchrun oracle comparison of every sharded mode (+ fake-rank tests)
cd $GRAFT_REPO_ROOT
o=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1 || { tail -20 $o/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_multigpu_gpu.py tests/test_exchange_gpu.py -q -x -p no:cacheprovider > $o/pytest_multi.log 2>&1; echo "multi pytest rc=$?"; tail -30 $o/pytest_multi.log
