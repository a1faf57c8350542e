# N = 4 fused: per-rank times with the single node-wide clock sampler, 6 runs; then N = 1 twice
cd $GRAFT_REPO_ROOT
o=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1 || { tail -20 $o/build.log; exit 1; }
for i in 1 2 3 4 5 6; do
GAR_BENCH_PER_RANK=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29580+i)) bench.py --gpus 4 --steps 20 --warmup 5 > $o/r2_skew_$i.log 2>&1
echo "$i rc=$?"
done
for i in 7 8; do timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $o/r2_skew_$i.log 2>&1; echo "$i rc=$?"; done
