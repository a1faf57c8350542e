#!/bin/bash
# Build experiment variants of libgar (tools only), swapping one Gram source:
#   tools/gram_exp.sh NAME SRC [nvcc -D flags...]   ->  libgar_NAME.so
# SRC replaces the product object of the same basename (gram_tc.o for
# gram_tc.cu or an experiments/*.cu copy of it, gram_f16.o for gram_f16.cu).
set -e
name=$1; src=$(realpath $2); shift 2
base=$(basename $src .cu); base=${base%%_r1}; base=${base%%_tf32}
case $base in gram_f16*) obj=gram_f16.o ;; gram_tc*) obj=gram_tc.o ;; *) obj=$base.o ;; esac
cd /root/repo/paper_2010_05888_b200
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  --expt-relaxed-constexpr -I csrc -I ../include "$@" -c $src -o /tmp/gram_$name.o
objs=$(ls _build/*.o | grep -v "/$obj\$")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o libgar_$name.so $objs /tmp/gram_$name.o -lcuda
