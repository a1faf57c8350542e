# CUDA-core Gram, two pair chunks (n = 16..22): coordinate pairs per lane and stage, A/B
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
NS="16 17 19 22"
for rep in 1 2; do
for v in prod st3 st4; do
  if [ $v = prod ]; then unset GAR_LIB_VARIANT; else export GAR_LIB_VARIANT=$v; fi
  timeout 300 python tools/gram_time.py $NS 2>&1 | tail -1
done; done
