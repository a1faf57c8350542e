# CUDA-core Gram with two pair chunks at 4 coordinate pairs per lane and stage: parity + sweeps
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 300 python tools/gram_time.py 16 17 19 20 22 2>&1 | tail -1
timeout 300 python tools/gram_time.py --bf16 16 19 22 2>&1 | tail -1
timeout 600 python tools/check_gram.py 2>&1 | sed -n 10,14p
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/cck4_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/cck4_pytest.log
timeout 600 python tools/sweep.py > gpurun_out/cck4_sweep_f32.md 2>&1; echo "sweep rc=$?"; head -8 gpurun_out/cck4_sweep_f32.md
timeout 600 python tools/sweep.py --bf16 > gpurun_out/cck4_sweep_bf16.md 2>&1; echo "sweep bf16 rc=$?"; head -8 gpurun_out/cck4_sweep_bf16.md
