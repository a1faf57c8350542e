#!/bin/bash
# Build experiment variants of libgar (tools only), recompiling one coordinate
# instantiation unit with extra flags:
#   tools/coord_exp.sh NAME UNIT [nvcc -D flags...]   ->  libgar_NAME.so
set -e
name=$1; unit=$2; shift 2
cd /root/repo/paper_2010_05888_b200
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -Xptxas -v --expt-relaxed-constexpr -I csrc -I ../include "$@" -c csrc/$unit.cu -o /tmp/coord_$name.o 2> /tmp/coord_$name.log
objs=$(ls _build/*.o | grep -v "/$unit.o\$")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o libgar_$name.so $objs /tmp/coord_$name.o -lcuda
