#!/usr/bin/env bash
# run ab_sweep.py for each ab/*.so given (names without .so)
tag=$1; shift
out=gpurun_out/$tag; mkdir -p $out
for v in "$@"; do
  CRB_LIB=ab/$v.so timeout 120 python scripts/ab_sweep.py 25 3 >> $out/ab.txt 2>&1
done
cat $out/ab.txt
