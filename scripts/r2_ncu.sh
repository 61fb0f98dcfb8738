#!/usr/bin/env bash
# one ncu --set full capture of the cfg 2 sweep at an early iteration (default 13)
set -u
tag=${1:-r2d}; skip=${2:-12}; cfg=${3:-cfg2}
out=gpurun_out/$tag; mkdir -p $out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_mma_kernel \
  --launch-skip $skip -c 1 -o $out/sweep_$cfg -f \
  python bench.py --config $cfg --steps $((skip+5)) --warmup 3 --no-cpu-baseline --no-extras > $out/ncu.log 2>&1
echo "ncu exit $?"; tail -3 $out/ncu.log
