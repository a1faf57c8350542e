#!/bin/bash
# Build libgar here first; only if that succeeds, run <script> on a GPU box.
#   tools/gpu.sh tools/gpu_xxx.sh [gpurun options...]
set -e
cd /root/repo
python paper_2010_05888_b200/build.py > /tmp/build_check.log 2>&1 || { echo "BUILD FAILED"; grep -E " error" /tmp/build_check.log | head; exit 1; }
script=$1; shift
exec timeout 4800 /usr/local/graft/bin/gpurun "$@" -- "bash $script"
