# converter preload of a whole raw stage: A/B on the tensor-core Gram (NP = 16 / 32), accuracy
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
NS="13 16 19 27 31"
for rep in 1 2; do
GAR_GRAM_CC=0 timeout 300 python tools/gram_time.py $NS 2>&1 | tail -1
GAR_LIB_VARIANT=pre0 GAR_GRAM_CC=0 timeout 300 python tools/gram_time.py $NS 2>&1 | tail -1
done
GAR_GRAM_CC=0 timeout 600 python tools/check_gram.py 2>&1 | tail -6
