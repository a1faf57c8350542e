cd $GRAFT_REPO_ROOT
for wl in sweep:35 sweep:47 sweep:63; do for rep in 1 2; do
timeout 300 python tools/ab_step.py $wl 2>&1 | tail -1
GAR_COORD_LOADER=tma timeout 300 python tools/ab_step.py $wl 2>&1 | tail -1
for v in w64a w64b; do GAR_COORD_LOADER=tma GAR_LIB_VARIANT=$v timeout 300 python tools/ab_step.py $wl 2>&1 | tail -1; done
done; done
