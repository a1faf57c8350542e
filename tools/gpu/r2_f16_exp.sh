# gram_f16 bottleneck attribution: GRAM16_EXP bit-mask variants (tools/gram_exp.sh), one Gram pass per n
cd $GRAFT_REPO_ROOT
o=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1 || { tail -20 $o/build.log; exit 1; }
V="18 26 27 59 63 8 34"
for x in $V; do bash tools/gram_exp.sh e$x paper_2010_05888_b200/csrc/gram_f16.cu -DGRAM16_EXP=$x > $o/exp_build_$x.log 2>&1 || { tail $o/exp_build_$x.log; exit 1; }; done
NS="19 31 35"
GAR_GRAM=tf32 timeout 300 python tools/gram_time.py $NS 2>&1 | tail -1
timeout 300 python tools/gram_time.py $NS 2>&1 | tail -1
for x in $V; do GAR_LIB_VARIANT=e$x timeout 300 python tools/gram_time.py $NS 2>&1 | tail -1; done
