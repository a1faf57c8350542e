cd $GRAFT_REPO_ROOT
for wl in C3 sweep:11 sweep:23 sweep:35 sweep:47; do for rep in 1 2; do
timeout 300 python tools/ab_step.py $wl 2>&1 | tail -1
GAR_LIB_VARIANT=pp timeout 300 python tools/ab_step.py $wl 2>&1 | tail -1
done; done
