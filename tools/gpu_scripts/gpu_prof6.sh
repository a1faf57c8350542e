cd $GRAFT_REPO_ROOT
NCU=/usr/local/cuda/bin/ncu
timeout 900 python bench.py > gpurun_out/f6_bench.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/f6_ref.log 2>&1; echo "ref rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/f6_short.log 2>&1 && \
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f6_launches.csv $CMD > gpurun_out/f6_ncu_launch.log 2>&1
echo "launch rc=$?"
timeout 300 python tools/prof_step.py > gpurun_out/f6_plain.log 2>&1 && \
timeout 1500 $NCU --set full --clock-control none --import-source on -k "regex:gram_tc|coord_select|coord_ldg|copy_row" -s 9 -c 9 -o gpurun_out/f6_full python tools/prof_step.py > gpurun_out/f6_ncu_full.log 2>&1
echo "full rc=$?"
