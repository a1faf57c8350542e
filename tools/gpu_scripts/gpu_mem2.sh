cd $GRAFT_REPO_ROOT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/membench2 tools/membench2.cu && timeout 600 /tmp/membench2 > gpurun_out/m2_membench.log 2>&1
echo "rc=$?" >> gpurun_out/m2_membench.log
for wl in C1 C2 C3; do timeout 300 python tools/ab_step.py $wl >> gpurun_out/m2_ab.log 2>&1; done
