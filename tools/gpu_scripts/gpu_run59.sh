cd $GRAFT_REPO_ROOT
for L in tma ldg; do for wl in sweep:7 sweep:11 sweep:19 sweep:23 sweep:27; do GAR_COORD_LOADER=$L timeout 300 python tools/ab_step.py $wl >> gpurun_out/r59.log 2>&1; done; done
