# Gram bottleneck attribution at NP = 32 for fp32 and bf16 rows (GRAM_EXP variants, results wrong by construction)
cd $GRAFT_REPO_ROOT
NS="19 27 31"
for v in prod exp1 exp3; do
  if [ $v = prod ]; then unset GAR_LIB_VARIANT; else export GAR_LIB_VARIANT=$v; fi
  GAR_GRAM_CC=0 timeout 300 python tools/gram_time.py $NS 2>&1 | tail -1
  GAR_GRAM_CC=0 timeout 300 python tools/gram_time.py --bf16 $NS 2>&1 | tail -1
done
