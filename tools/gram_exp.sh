#!/bin/bash
# Build experiment variants of libgar (tools only), swapping gram_tc.cu:
#   tools/gram_exp.sh NAME SRC [nvcc -D flags...]   ->  libgar_NAME.so
set -e
name=$1; src=$(realpath $2); shift 2
cd /root/repo/paper_2010_05888_b200
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  --expt-relaxed-constexpr -I csrc -I ../include "$@" -c $src -o /tmp/gram_$name.o
objs=$(ls _build/*.o | grep -v '/gram_tc.o$')
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o libgar_$name.so $objs /tmp/gram_$name.o -lcuda
