#!/usr/bin/env bash
# fp64 pipe microbenchmark + cfg 2 sweep captures: one ncu --set full at an early
# iteration, and the DRAM bytes / duration of every sweep launch of the bench's
# timed region (--steps 20 --warmup 5: launches 6..25)
set -u
tag=${1:-r2p}; skip=${2:-12}
out=gpurun_out/$tag; mkdir -p $out
timeout 120 ./scripts/micro/fp64_tput > $out/fp64_tput.txt 2>&1; cat $out/fp64_tput.txt
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --clock-control none -k regex:sweep_mma_kernel --csv --log-file $out/timed_sweeps.csv \
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extras > $out/timed_ncu.log 2>&1
echo "timed ncu exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_mma_kernel \
  --launch-skip $skip -c 1 -o $out/sweep_cfg2 -f \
  python bench.py --steps $((skip+5)) --warmup 3 --no-cpu-baseline --no-extras > $out/ncu.log 2>&1
echo "ncu exit $?"; tail -2 $out/ncu.log
