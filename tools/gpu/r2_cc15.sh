# CUDA-core Gram up to n = 15: time per pass against the tensor cores, accuracy, parity suite, C5 sweep
cd $GRAFT_REPO_ROOT
o=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1 || { tail -20 $o/build.log; exit 1; }
NS="${NS:-7 11 12 13 14 15 16}"
timeout 300 python tools/gram_time.py $NS 2>&1 | tail -1
GAR_GRAM_CC=0 timeout 300 python tools/gram_time.py $NS 2>&1 | tail -1
timeout 600 python tools/check_gram.py 2>&1 | head -12
timeout 1500 python -m pytest tests -m gpu -x -q > $o/cc15_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $o/cc15_pytest.log
timeout 600 python tools/sweep.py > $o/cc15_sweep_f32.md 2>&1; echo "sweep rc=$?"; head -8 $o/cc15_sweep_f32.md
timeout 600 python tools/sweep.py --bf16 > $o/cc15_sweep_bf16.md 2>&1; echo "sweep bf16 rc=$?"; head -8 $o/cc15_sweep_bf16.md
