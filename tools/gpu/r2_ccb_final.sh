# register-blocked CUDA-core Gram for n = 33..36 in the product: timing, accuracy, parity suite, C5 sweep
cd $GRAFT_REPO_ROOT
o=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1 || { tail -20 $o/build.log; exit 1; }
timeout 300 python tools/gram_time.py 32 33 34 35 36 37 2>&1 | tail -1
timeout 300 python tools/gram_time.py --bf16 33 35 36 2>&1 | tail -1
GAR_GRAM_CC=0 timeout 300 python tools/gram_time.py --bf16 33 35 36 2>&1 | tail -1
timeout 600 python tools/check_gram.py 2>&1 | grep "n=33\|n=32\|high"
timeout 600 python tools/check_gram_bf16.py 2>&1 | grep "n=33\|worst"
timeout 1500 python -m pytest tests -m gpu -x -q > $o/ccbf_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $o/ccbf_pytest.log
timeout 600 python tools/sweep.py > $o/ccbf_sweep_f32.md 2>&1; echo "sweep rc=$?"; sed -n 3,13p $o/ccbf_sweep_f32.md
timeout 600 python tools/sweep.py --bf16 > $o/ccbf_sweep_bf16.md 2>&1; echo "sweep bf16 rc=$?"; sed -n 10,12p $o/ccbf_sweep_bf16.md
