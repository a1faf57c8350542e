# C5 sweep (fp32 and bf16) with an nvidia-smi clock record alongside
cd $GRAFT_REPO_ROOT
o=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1 || { tail -20 $o/build.log; exit 1; }
nvidia-smi --query-gpu=timestamp,clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_event_reasons.active --format=csv,noheader -lms 500 > $o/r2_sweep_clocks.csv 2>&1 &
SMI=$!
timeout 900 python tools/sweep.py > $o/r2_sweep_f32.md 2>&1; echo "sweep f32 rc=$?"
timeout 900 python tools/sweep.py --bf16 > $o/r2_sweep_bf16.md 2>&1; echo "sweep bf16 rc=$?"
kill $SMI
cat $o/r2_sweep_f32.md | head -20; cat $o/r2_sweep_bf16.md | head -20
