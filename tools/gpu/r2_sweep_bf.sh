cd $GRAFT_REPO_ROOT
o=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1 || { tail -20 $o/build.log; exit 1; }
timeout 900 python tools/sweep.py --bf16 > $o/r2_sweep_bf16.md 2>&1; echo "sweep bf16 rc=$?"
head -18 $o/r2_sweep_bf16.md
timeout 900 python -m pytest tests/test_bf16_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -2
