#!/usr/bin/env bash
out=gpurun_out/${1:-cwscan}; mkdir -p $out
for n in 1 3 5 8 12 16 24 32; do
  for v in all15 all11; do
    CRB_LIB=ab/$v.so timeout 300 python scripts/ab_sweep.py 25 2 10000 $n 2>&1 | sed "s/^/n=$n /" | cut -c1-70 >> $out/scan.txt
  done
done
cat $out/scan.txt
