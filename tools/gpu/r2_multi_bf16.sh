# 2-GPU bench variants: bf16 rows (replicated output, NCCL exchange), fp32 with --exchange nccl, sharded
cd $GRAFT_REPO_ROOT
o=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1 || { tail -20 $o/build.log; exit 1; }
i=0
for args in "--dtype bf16" "--exchange nccl" "--output sharded" "--impl reference"; do
i=$((i+1))
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29590+i)) bench.py --gpus 2 --steps 10 --warmup 3 $args > $o/r2_mb_$i.log 2>&1
echo "[$args] rc=$? $(grep '^{' $o/r2_mb_$i.log | cut -c1-330)"
done
