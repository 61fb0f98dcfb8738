#!/usr/bin/env bash
# DRAM bytes and duration of every sweep launch of the default driver bench
# command's timed region (--steps 20 --warmup 5: sweep launches 6..25)
set -u
out=gpurun_out/${1:-r2t}; mkdir -p $out
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --clock-control none -k regex:sweep_mma_kernel --csv --log-file $out/timed_sweeps.csv \
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extras > $out/timed_ncu.log 2>&1
echo "timed ncu exit $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $out/launches.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extras \
  > $out/launches_ncu.log 2>&1
echo "launch list exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_mma_kernel \
  --launch-skip 12 -c 1 -o $out/sweep_cfg2_it13 -f \
  python bench.py --steps 17 --warmup 3 --no-cpu-baseline --no-extras > $out/ncu_full.log 2>&1
echo "ncu full exit $?"
