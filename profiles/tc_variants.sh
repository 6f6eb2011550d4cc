#!/bin/bash
# Build variants of libmprk_b200.so that differ only in the folded tcgen05
# contraction's compile-time pipeline shape (tensor_tc.cu TF_* macros), for
# A/B timing with profiles/tc_variants.py on the GPU box.
#   profiles/tc_variants.sh name "-DTF_CS=3 -DTF_RS_N=3" [name2 "flags2" ...]
set -e
cd "$(dirname "$0")/.."
PKG=paper_2412_16638_b200
OBJS=$(ls $PKG/build/*.o | grep -v tensor_tc.cu.o)
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  d=profiles/_variants/$name; mkdir -p $d
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC \
    --expt-relaxed-constexpr -Iinclude $flags -c $PKG/csrc/tensor_tc.cu -o $d/tensor_tc.o
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $d/libmprk_b200.so $OBJS $d/tensor_tc.o \
    -Xlinker -z,defs -lcudart_static -lrt -ldl -lpthread
  echo "$name: $flags" > $d/flags.txt
done
