#!/usr/bin/env bash
# ab_sweep.py at a given N, n for each ab/*.so: ab_run_n.sh tag N n names...
tag=$1; N=$2; n=$3; shift 3
out=gpurun_out/$tag; mkdir -p $out
for v in "$@"; do CRB_LIB=ab/$v.so timeout 300 python scripts/ab_sweep.py 25 2 $N $n >> $out/ab.txt 2>&1; done
cat $out/ab.txt
