cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/f8_pytest.log 2>&1; tail -2 gpurun_out/f8_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/f8_smoke.log 2>&1; tail -1 gpurun_out/f8_smoke.log
timeout 900 python bench.py > gpurun_out/f8_bench.log 2>&1; echo "bench rc=$?"; grep '^{' gpurun_out/f8_bench.log | tail -1 | cut -c1-300
