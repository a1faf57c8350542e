# tf32 Gram: TMEM drain window (FLUSH) per NP and padded-column skip; one pass per n, variants via gram_exp.sh
cd $GRAFT_REPO_ROOT
o=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1 || { tail -20 $o/build.log; exit 1; }
for v in "f32_3:-DGRAM_FLUSH32=3" "f32_4:-DGRAM_FLUSH32=4" "f64_2:-DGRAM_FLUSH64=2" "f64_6:-DGRAM_FLUSH64=6" "f64_8:-DGRAM_FLUSH64=8"; do
  name=${v%%:*}; flag=${v#*:}
  bash tools/gram_exp.sh $name paper_2010_05888_b200/csrc/gram_tc.cu $flag > $o/exp_$name.log 2>&1 || { tail $o/exp_$name.log; exit 1; }
done
NS="19 23 31 35 39 47 55 63"
timeout 300 python tools/gram_time.py $NS 2>&1 | tail -1 | tee -a $o/flush.log
for name in f32_3 f32_4 f64_2 f64_6 f64_8; do GAR_LIB_VARIANT=$name timeout 300 python tools/gram_time.py $NS 2>&1 | tail -1 | tee -a $o/flush.log; done

