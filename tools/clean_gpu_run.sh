#!/bin/bash
# The driver's round-end sequence, reproduced on a GPU box from a CLEAN copy of
# the snapshot (no libgar.so, no _build/, no oracle .so):
#   build() -> smoke() -> pytest -m gpu -x -q -> bench.py --gpus 1 --steps 20 --warmup 5
# Logs with wall times go to gpurun_out/clean_<tag>.log.
#   gpurun --timeout 2400 -- 'bash tools/clean_gpu_run.sh r2a'
tag=${1:-run}
src=${GRAFT_REPO_ROOT:-/root/repo}
out=$src/gpurun_out/clean_$tag.log
mkdir -p $src/gpurun_out
dst=/tmp/clean_$tag
rm -rf $dst && mkdir -p $dst
( cd $src && tar --exclude=./gpurun_out --exclude='*.so' --exclude='*.o' --exclude=./paper_2010_05888_b200/_build \
    --exclude=./baseline -cf - . ) | ( cd $dst && tar -xf - )
cd $dst
{
echo "== clean copy at $dst: $(find . -name '*.so' | wc -l) .so files, $(nproc) cores"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
t0=$(date +%s)
timeout 900 python -c "import __graft_entry__ as g; g.build()" > /tmp/build.log 2>&1; echo "build rc=$? $(( $(date +%s)-t0 )) s"; tail -2 /tmp/build.log
t0=$(date +%s)
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3; echo "smoke rc=${PIPESTATUS[0]} $(( $(date +%s)-t0 )) s"
t0=$(date +%s)
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > /tmp/pytest.log 2>&1; echo "pytest -m gpu rc=$? $(( $(date +%s)-t0 )) s"; tail -3 /tmp/pytest.log
t0=$(date +%s)
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > /tmp/bench.log 2>&1; echo "bench rc=$? $(( $(date +%s)-t0 )) s"; tail -c 6000 /tmp/bench.log
} > $out 2>&1
cp /tmp/pytest.log $src/gpurun_out/clean_${tag}_pytest.log
cat $out
