cd $GRAFT_REPO_ROOT
for wl in C3 C4 sweep:23 sweep:27 sweep:15; do for rep in 1 2; do
timeout 300 python tools/ab_step.py $wl 2>&1 | tail -1
for v in bw24 bw20; do GAR_COORD_LOADER=tma GAR_LIB_VARIANT=$v timeout 300 python tools/ab_step.py $wl 2>&1 | tail -1; done
done; done
