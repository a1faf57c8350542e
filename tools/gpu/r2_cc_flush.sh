# CUDA-core Gram n <= 15: stages summed in fp32 per flush (8 / 16 / 32), A/B + accuracy
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
NS="8 11 12 13 15"
for rep in 1 2; do
for v in prod fl16 fl32; do
  if [ $v = prod ]; then unset GAR_LIB_VARIANT; else export GAR_LIB_VARIANT=$v; fi
  timeout 300 python tools/gram_time.py $NS 2>&1 | tail -1
done; done
GAR_LIB_VARIANT=fl32 timeout 600 python tools/check_gram.py 2>&1 | sed -n 3,9p
