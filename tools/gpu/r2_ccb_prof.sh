# ncu --set full of one register-blocked CUDA-core Gram pass (n = $1, default 31)
cd $GRAFT_REPO_ROOT
o=gpurun_out
N=${1:-31}
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1 || { tail -20 $o/build.log; exit 1; }
timeout 300 python tools/gram_time.py $N 2>&1 | tail -1
GAR_GRAM_CC=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:${KREGEX:-gram_ccb} -s 2 -c 1 -o /tmp/ccb -f python tools/gram_one.py $N > $o/ccb_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/ccb.ncu-rep --page source --csv --print-source cuda,sass > /tmp/ccb_src.csv 2>&1
python tools/ncu_lines.py /tmp/ccb_src.csv 30 > $o/ccb_lines.txt 2>&1
ncu -i /tmp/ccb.ncu-rep --page details --csv > $o/ccb_details.csv 2>&1
ncu -i /tmp/ccb.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__warps_active.avg.per_cycle_active,dram__bytes_read.sum,launch__grid_size,launch__registers_per_thread > $o/ccb_raw.csv 2>&1
cat $o/ccb_lines.txt | cut -c1-220; cat $o/ccb_raw.csv | tail -1 | cut -c1-800
grep -i "stall\|warp cycles\|issued" $o/ccb_details.csv | cut -c1-250 | head -40
ncu -i /tmp/ccb.ncu-rep --page raw --csv --metrics regex:smsp__average_warps_issue_stalled_.*_per_issue_active.ratio > $o/ccb_stalls.csv 2>&1
python3 - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/ccb_stalls.csv")))
h, v = rows[0], rows[-1]
xs = sorted(((float(b), a) for a, b in zip(h, v) if a.startswith("smsp__average") and b.replace('.', '', 1).isdigit()), reverse=True)
for val, name in xs[:14]:
    print(f"{val:7.3f} {name}")
PY
