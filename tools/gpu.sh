#!/bin/bash
# Run <script> on a B200 via gpurun.  Nothing is prebuilt here: the box builds
# libgar.so from source exactly as the driver's clean checkout does.
#   tools/gpu.sh tools/gpu/xxx.sh [gpurun options...]
set -e
cd /root/repo
script=$1; shift
exec timeout 4800 /usr/local/graft/bin/gpurun "$@" -- "bash $script"
