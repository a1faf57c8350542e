cd $GRAFT_REPO_ROOT
for L in tma ldg; do for wl in C3 sweep:15 sweep:47; do GAR_COORD_LOADER=$L timeout 300 python tools/ab_step.py $wl >> gpurun_out/r58.log 2>&1; done; done
