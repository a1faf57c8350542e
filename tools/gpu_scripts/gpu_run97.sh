cd $GRAFT_REPO_ROOT
for L in tma ldg; do for wl in C3 C2; do GAR_COORD_LOADER=$L timeout 300 python tools/phase_time.py $wl >> gpurun_out/r97.log 2>&1; done; done
