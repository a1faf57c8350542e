# ncu --set full of one bf16 and one fp32 C3 step (coordinate kernels + Gram); raw metrics exported
# on the box as CSV (the reports themselves exceed gpurun's 64 MiB return limit)
cd $GRAFT_REPO_ROOT
o=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1 || { tail -20 $o/build.log; exit 1; }
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed,launch__registers_per_thread,launch__grid_size,launch__block_size
for v in "bf16:bf16:9" "f32::9"; do
  tag=${v%%:*}; rest=${v#*:}; arg=${rest%%:*}; cnt=${rest#*:}
  timeout 1200 ncu --set full --clock-control none -k regex:'gram_tc|coord_select|copy_row' \
    --launch-skip $cnt -c $cnt -o /tmp/r2_$tag -f python tools/prof_step.py C3 $arg > $o/r2_${tag}_ncu.log 2>&1
  echo "ncu $tag rc=$?"
  ncu -i /tmp/r2_$tag.ncu-rep --page raw --csv --metrics $M > $o/r2_${tag}_metrics.csv 2>&1
done
