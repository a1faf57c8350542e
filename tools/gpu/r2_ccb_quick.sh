# CUDA-core Gram A/B: time per pass (CC product / tensor cores / variants), accuracy
cd $GRAFT_REPO_ROOT
o=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1 || { tail -20 $o/build.log; exit 1; }
NS="${NS:-13 16 19 24 27 31 35 40}"
GAR_GRAM_CC=1 timeout 300 python tools/gram_time.py $NS 2>&1 | tail -1
GAR_GRAM_CC=0 timeout 300 python tools/gram_time.py $NS 2>&1 | tail -1
for v in $VARIANTS; do GAR_LIB_VARIANT=$v GAR_GRAM_CC=1 timeout 300 python tools/gram_time.py $NS 2>&1 | tail -1; done
timeout 600 python tools/check_gram.py 2>&1 | tail -8
