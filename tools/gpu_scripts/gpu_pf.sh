cd $GRAFT_REPO_ROOT
for wl in C3 C4 sweep:7 sweep:11 sweep:19 sweep:23 sweep:35 sweep:47 sweep:63; do for rep in 1 2; do
timeout 300 python tools/ab_step.py $wl 2>&1 | tail -1
GAR_LIB_VARIANT=pf timeout 300 python tools/ab_step.py $wl 2>&1 | tail -1
done; done
