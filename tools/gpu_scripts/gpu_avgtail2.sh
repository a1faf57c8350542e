cd $GRAFT_REPO_ROOT
for n in 7 11 15 35 63; do for rep in 1 2; do
GAR_LIB_VARIANT=serial timeout 300 python tools/ab_step.py sweep:$n 2>&1 | tail -1 | grep -o '"workload.*"median": [0-9.]*'
timeout 300 python tools/ab_step.py sweep:$n 2>&1 | tail -1 | grep -o '"workload.*"median": [0-9.]*'
done; done
