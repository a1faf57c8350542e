# tf32 Gram at NP = 64: ring geometry variants (op stages, raw tiles per stage, raw stages, producer warps)
cd $GRAFT_REPO_ROOT
o=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1 || { tail -20 $o/build.log; exit 1; }
V="o3s3:-DGRAM64_OPS=3+-DGRAM64_RAW_SUB=3 s2r3:-DGRAM64_RAW_SUB=2+-DGRAM64_RAW_STAGES=3 o3s2:-DGRAM64_OPS=3+-DGRAM64_RAW_SUB=2 o4s2:-DGRAM64_OPS=4+-DGRAM64_RAW_SUB=2"
for v in $V; do name=${v%%:*}; flags=$(echo ${v#*:} | tr '+' ' ')
  bash tools/gram_exp.sh $name paper_2010_05888_b200/csrc/gram_tc.cu $flags > $o/exp_$name.log 2>&1 || { tail $o/exp_$name.log; exit 1; }; done
NS="35 47 63"
rm -f $o/np64.log
timeout 300 python tools/gram_time.py $NS 2>&1 | tail -1 | tee -a $o/np64.log
for v in $V; do name=${v%%:*}; GAR_LIB_VARIANT=$name timeout 300 python tools/gram_time.py $NS 2>&1 | tail -1 | tee -a $o/np64.log; done
