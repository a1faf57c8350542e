# bf16 row: parity tests first, then the whole -m gpu suite, then the benches.
cd $GRAFT_REPO_ROOT
o=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1 || { tail -20 $o/build.log; exit 1; }
timeout 900 python -m pytest tests/test_bf16_gpu.py tests/test_bench_contract.py -q -x -p no:cacheprovider > $o/pytest_bf16.log 2>&1; echo "bf16 pytest rc=$?"; tail -15 $o/pytest_bf16.log
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider > $o/pytest_all.log 2>&1; echo "all pytest rc=$?"; tail -6 $o/pytest_all.log
timeout 600 python bench.py --steps 10 --warmup 3 > $o/bench.log 2>&1; echo "bench rc=$?"; tail -c 600 $o/bench.log
timeout 600 python bench.py --steps 10 --warmup 3 --dtype bf16 > $o/bench_bf16.log 2>&1; echo "bench bf16 rc=$?"; tail -c 3000 $o/bench_bf16.log
