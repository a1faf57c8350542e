# ncu of the fused Gram + selection kernel at C2 (Krum)
cd $GRAFT_REPO_ROOT
o=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1 || { tail -20 $o/build.log; exit 1; }
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gram_cc -s 2 -c 1 -o /tmp/fz -f python tools/krum_one.py C2 krum > $o/fz_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/fz.ncu-rep --page source --csv --print-source cuda,sass > /tmp/fz_src.csv 2>&1
python tools/ncu_lines.py /tmp/fz_src.csv 25 > $o/fz_lines.txt 2>&1
ncu -i /tmp/fz.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,launch__registers_per_thread,launch__grid_size > $o/fz_raw.csv 2>&1
cut -c1-220 $o/fz_lines.txt; tail -1 $o/fz_raw.csv
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/fz_launches.csv python tools/krum_one.py C2 krum > /dev/null 2>&1
grep -E "gram|select|copy_row|memset" $o/fz_launches.csv | tail -8 | cut -c1-300
