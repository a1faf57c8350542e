# proxy-fence cost in the tensor-core Gram converters (GRAM_EXP=5 skips it; results wrong by construction)
cd $GRAFT_REPO_ROOT
NS="19 27 31 35 63"
for v in prod exp5 exp1; do
  if [ $v = prod ]; then unset GAR_LIB_VARIANT; else export GAR_LIB_VARIANT=$v; fi
  GAR_GRAM_CC=0 timeout 300 python tools/gram_time.py $NS 2>&1 | tail -1
done
