# Gram A/B with attribution variants + one ncu capture of the product kernel at n = 31 and 47.
cd $GRAFT_REPO_ROOT
o=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1 || { tail -20 $o/build.log; exit 1; }
bash tools/gram_exp.sh r1 tools/experiments/gram_tc_tf32_r1.cu > $o/gram_exp.log 2>&1 || { tail $o/gram_exp.log; exit 1; }
bash tools/gram_exp.sh nomma paper_2010_05888_b200/csrc/gram_tc.cu -DGRAM_EXP=1 >> $o/gram_exp.log 2>&1
bash tools/gram_exp.sh nost paper_2010_05888_b200/csrc/gram_tc.cu -DGRAM_EXP=2 >> $o/gram_exp.log 2>&1
bash tools/gram_exp.sh sub2 paper_2010_05888_b200/csrc/gram_tc.cu -DGRAM_NP64_SUB=2 >> $o/gram_exp.log 2>&1
NS="7 11 15 19 31 35 47 63"
for v in prod r1 nomma nost sub2; do
  if [ $v = prod ]; then timeout 600 python tools/gram_time.py $NS 2>&1 | tail -1
  else GAR_LIB_VARIANT=$v timeout 600 python tools/gram_time.py $NS 2>&1 | tail -1; fi
done
timeout 600 python tools/check_gram.py > $o/check_gram.log 2>&1; echo "check_gram rc=$?"; tail -3 $o/check_gram.log
for n in 31 47; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gram_tc -s 2 -c 1 -o $o/gram_n$n -f python tools/gram_one.py $n > $o/gram_ncu_$n.log 2>&1
echo "ncu n=$n rc=$?"
done
