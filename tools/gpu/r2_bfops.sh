# bf16 rows: Gram with bf16 hi/lo operands (kind::f16) vs the tf32 path on widened values; accuracy; parity suite
cd $GRAFT_REPO_ROOT
o=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1 || { tail -20 $o/build.log; exit 1; }
timeout 600 python tools/check_gram_bf16.py 2>&1 | tail -14
GAR_LIB_VARIANT=bfops0 timeout 600 python tools/check_gram_bf16.py 2>&1 | tail -3
NS="23 27 31 35 47 63"
timeout 300 python tools/gram_time.py --bf16 $NS 2>&1 | tail -1
GAR_LIB_VARIANT=bfops0 timeout 300 python tools/gram_time.py --bf16 $NS 2>&1 | tail -1
timeout 300 python tools/gram_time.py $NS 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -x -q > $o/bfops_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $o/bfops_pytest.log
