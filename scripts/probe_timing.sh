#!/usr/bin/env bash
tag=$1; shift
out=gpurun_out/$tag; mkdir -p $out
for v in "$@"; do
  CRB_LIB=ab/$v.so timeout 120 python scripts/ab_sweep.py 14 1 > $out/$v.txt 2>&1
  echo "== $v"; grep -c probe $out/$v.txt; tail -1 $out/$v.txt | cut -c1-120
done
