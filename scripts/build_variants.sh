#!/usr/bin/env bash
# build n=10-only variants of one source (SRC, default sweep_mma.cu) in parallel:
# ab/<name>.so for each "name:flags" argument
set -e
B=build/cvxreg_b200
SRC=${SRC:-sweep_mma.cu}
EXCL=${EXCL:-$SRC}
objs=$(ls $B/*.o | grep -v $EXCL.o)
# NLIST=k: kernels for one n only (fast builds); NLIST=all: every n
NLIST=${NLIST:-10}
if [ "$NLIST" = all ]; then NDEF=""; else NDEF="-DCRB_N_LIST=$NLIST"; fi
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  ( /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
      -Xcompiler -fPIC -Xcompiler -ffp-contract=off -Iinclude $NDEF $flags \
      -c paper_1407_7220_b200/csrc/$SRC -o /tmp/v_$name.o && \
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ab/$name.so \
      /tmp/v_$name.o $objs -lnccl -lcudart_static -lrt -lpthread -ldl && echo built $name ) &
done
wait
