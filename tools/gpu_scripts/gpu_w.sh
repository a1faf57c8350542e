cd $GRAFT_REPO_ROOT
for wl in C3 sweep:23; do for rep in 1 2; do
timeout 300 python tools/ab_step.py $wl 2>&1 | tail -1
for v in w20 w24 w12; do GAR_LIB_VARIANT=$v timeout 300 python tools/ab_step.py $wl 2>&1 | tail -1; done
done; done
