#!/bin/bash
# Build experiment variants of libgar (tools only), recompiling coordinate
# instantiation units with extra flags:
#   tools/coord_exp.sh NAME UNIT[,UNIT...] [nvcc -D flags...]   ->  libgar_NAME.so
set -e
name=$1; units=$2; shift 2
cd /root/repo/paper_2010_05888_b200
objs=$(ls _build/*.o)
extra=""
for unit in ${units//,/ }; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -Xptxas -v --expt-relaxed-constexpr -I csrc -I ../include "$@" -c csrc/$unit.cu -o /tmp/coord_${name}_$unit.o \
    2> /tmp/coord_${name}_$unit.log &
  objs=$(echo "$objs" | grep -v "/$unit.o\$")
  extra="$extra /tmp/coord_${name}_$unit.o"
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o libgar_$name.so $objs $extra -lcuda
