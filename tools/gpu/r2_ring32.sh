# NP = 32 ring geometry A/B: operand stages x tiles per raw stage
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
NS="19 27 31"
for rep in 1 2; do
for v in prod o2r4 o2r5 o2r6; do
  if [ $v = prod ]; then unset GAR_LIB_VARIANT; else export GAR_LIB_VARIANT=$v; fi
  GAR_GRAM_CC=0 timeout 300 python tools/gram_time.py $NS 2>&1 | tail -1
done
done
