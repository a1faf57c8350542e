# bench (no profiler) -> ncu launch list of the same command -> one ncu --set full
# capture of one step's kernels.  Usage: bash tools/gpu/profile.sh TAG [WORKLOAD]
cd $GRAFT_REPO_ROOT
tag=${1:-p}; wl=${2:-C3}; EXTRA=${3:-}
o=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1 || { tail -20 $o/build.log; exit 1; }
timeout 900 python bench.py --workload $wl --steps 20 --warmup 5 $EXTRA > $o/${tag}_bench.log 2>&1; echo "bench rc=$?"
tail -c 5000 $o/${tag}_bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/${tag}_launches.csv \
  python bench.py --workload $wl --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-variants $EXTRA > $o/${tag}_ncu_list.log 2>&1
echo "launch list rc=$?"
# one step = the last launches of the timed region; skip the warm-up steps (each step ~16 kernels)
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'gram_tc|coord_select|copy_row|select_kernel|gram_reduce' \
  --launch-skip 45 -c 15 -o $o/${tag}_full -f \
  python bench.py --workload $wl --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-variants $EXTRA > $o/${tag}_ncu_full.log 2>&1
echo "ncu full rc=$?"
ls -la $o/ | tail -8
