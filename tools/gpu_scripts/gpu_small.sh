cd $GRAFT_REPO_ROOT
for wl in sweep:7 sweep:11 sweep:15 sweep:19; do for rep in 1 2; do
timeout 300 python tools/ab_step.py $wl 2>&1 | tail -1
GAR_COORD_LOADER=tma timeout 300 python tools/ab_step.py $wl 2>&1 | tail -1
done; done
