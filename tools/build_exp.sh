#!/bin/bash
# Experiment builds of the fire kernel: _exp/libxlfuse_b200_<n>.so with -DFIRE_EXP=<n>
# (same objects otherwise).  Usage: tools/build_exp.sh 1 2 3
set -e
cd "$(dirname "$0")/.."
C=paper_2007_06000_b200/csrc
mkdir -p _exp
for n in "$@"; do
  /usr/local/cuda/bin/nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -DFIRE_EXP=$n \
    -c $C/kernels_fire.cu -o _exp/kernels_fire_$n.o &
done
wait
for n in "$@"; do
  objs=$(ls $C/build/*.o | grep -v kernels_fire.o)
  /usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -cudart static -o _exp/libxlfuse_b200_$n.so $objs _exp/kernels_fire_$n.o -lrt -ldl -lpthread
done
ls -la _exp
