cd $GRAFT_REPO_ROOT
for wl in C1 C2; do timeout 300 python tools/graph_latency.py $wl >> gpurun_out/r82.log 2>&1; done
