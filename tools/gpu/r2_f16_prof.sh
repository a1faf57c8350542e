# ncu --set full of one gram_f16 pass at n = 31 and n = 35 (tools/gram_one.py)
cd $GRAFT_REPO_ROOT
o=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1 || { tail -20 $o/build.log; exit 1; }
for n in 31 35; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gram_f16 -s 2 -c 1 -o $o/g16_n$n -f python tools/gram_one.py $n > $o/g16_ncu_$n.log 2>&1
echo "ncu n=$n rc=$?"
done
