# ncu --set full of the Gram kernel and the Bulyan selection at small d (fixed per-call costs)
cd $GRAFT_REPO_ROOT
o=gpurun_out
for k in gram_tc select_kernel; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 2 -c 1 -o /tmp/sp_$k -f python tools/gram_small_one.py > $o/sp_$k.log 2>&1; echo "ncu $k rc=$?"
ncu -i /tmp/sp_$k.ncu-rep --page source --csv --print-source cuda,sass > /tmp/sp_src.csv 2>&1
python tools/ncu_lines.py /tmp/sp_src.csv 22 | cut -c1-230
ncu -i /tmp/sp_$k.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active | tail -1 | cut -c1-300
done
