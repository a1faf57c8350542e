cd $GRAFT_REPO_ROOT
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $R --nproc-per-node 4 --master-port 29561 tools/check_fused.py C3 > gpurun_out/fmg_check4.log 2>&1; echo "check4 rc=$?"; tail -3 gpurun_out/fmg_check4.log
for N in 2 4; do
timeout 900 $R --nproc-per-node $N --master-port 2957$N bench.py --gpus $N > gpurun_out/fmg_bench_$N.log 2>&1; echo "bench$N rc=$?"; grep '^{' gpurun_out/fmg_bench_$N.log | tail -1 | cut -c1-400
timeout 600 $R --nproc-per-node $N --master-port 2958$N bench.py --gpus $N --impl reference > gpurun_out/fmg_ref_$N.log 2>&1; echo "ref$N rc=$?"; grep '^{' gpurun_out/fmg_ref_$N.log | tail -1 | cut -c1-200
done
