#!/usr/bin/env bash
# ncu --set full of one cfg2 sweep launch (iteration skip+1) for ab/<variant>.so
set -u
tag=$1; v=$2; skip=${3:-12}
out=gpurun_out/$tag; mkdir -p $out
CRB_LIB=ab/$v.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_mma_kernel \
  --launch-skip $skip -c 1 -o $out/sweep_$v -f python scripts/ab_sweep.py $((skip+2)) 1 > $out/ncu_$v.log 2>&1
echo "ncu $v exit $?"
