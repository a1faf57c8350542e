cd $GRAFT_REPO_ROOT
for wl in sweep:35 sweep:39 sweep:43 sweep:47; do for rep in 1 2; do
timeout 300 python tools/ab_step.py $wl 2>&1 | tail -1
for v in w48a w48b; do GAR_COORD_LOADER=tma GAR_LIB_VARIANT=$v timeout 300 python tools/ab_step.py $wl 2>&1 | tail -1; done
done; done
