cd $GRAFT_REPO_ROOT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/membench tools/membench.cu && timeout 600 /tmp/membench > gpurun_out/m1_membench.log 2>&1
echo "rc=$?" >> gpurun_out/m1_membench.log
