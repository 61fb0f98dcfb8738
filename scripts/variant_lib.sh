#!/usr/bin/env bash
# A/B helper: rebuild sweep_mma.cu with extra nvcc flags and link it with the
# other objects of the last in-tree build into <out.so> (e.g. -DCRB_WIDE_ABOVE=0).
#   bash scripts/variant_lib.sh out.so -DFLAG=...
set -e
out=$1; shift
B=build/cvxreg_b200
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC -Xcompiler -ffp-contract=off -Iinclude "$@" \
  -c paper_1407_7220_b200/csrc/sweep_mma.cu -o /tmp/variant_sweep_mma.o
objs=$(ls $B/*.o | grep -v sweep_mma.cu.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out" \
  /tmp/variant_sweep_mma.o $objs -lnccl -lcudart_static -lrt -lpthread -ldl
