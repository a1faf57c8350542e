cd $GRAFT_REPO_ROOT
for wl in sweep:51 sweep:55 sweep:59 sweep:63; do for rep in 1 2; do
timeout 300 python tools/ab_step.py $wl 2>&1 | tail -1
GAR_LIB_VARIANT=part24 timeout 300 python tools/ab_step.py $wl 2>&1 | tail -1
GAR_LIB_VARIANT=part40 timeout 300 python tools/ab_step.py $wl 2>&1 | tail -1
done; done
