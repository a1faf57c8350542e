cd $GRAFT_REPO_ROOT
o=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1 || { tail -20 $o/build.log; exit 1; }
GAR_GRAM_CC=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:gram_cc -s 2 -c 1 -o /tmp/cc11 -f python tools/gram_one.py 11 > $o/cc_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/cc11.ncu-rep --page source --csv --print-source cuda,sass > /tmp/cc_src.csv 2>&1
python tools/ncu_lines.py /tmp/cc_src.csv 25 > $o/cc_lines.txt 2>&1
ncu -i /tmp/cc11.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__warps_active.avg.per_cycle_active > $o/cc_raw.csv 2>&1
cat $o/cc_lines.txt | cut -c1-220; cat $o/cc_raw.csv | tail -1 | cut -c1-600
