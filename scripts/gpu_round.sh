#!/usr/bin/env bash
# One gpurun call: GPU tests, the default bench line, the reference arm, the
# launch list of a short bench and one `ncu --set full` sweep capture at
# iteration ~1000 of cfg 2 (the late, sparse regime the timed region sits in).
#   gpurun --timeout 2400 -- 'bash scripts/gpu_round.sh <tag> [tests|notests]'
set -u
tag=${1:-r}
tests=${2:-tests}
out=gpurun_out/$tag
mkdir -p "$out"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > "$out/gpu.txt" 2>&1
if [ "$tests" = tests ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > "$out/pytest_gpu.log" 2>&1
  echo "pytest exit $?" >> "$out/pytest_gpu.log"
  tail -3 "$out/pytest_gpu.log"
fi
timeout 600 python bench.py > "$out/bench_cfg2.json" 2> "$out/bench_cfg2.err"; echo "bench exit $?"
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > "$out/bench_reference.json" 2> "$out/bench_reference.err"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file "$out/launches.csv" python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extras \
  > "$out/ncu_launch.log" 2>&1; echo "launch list exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_mma_kernel \
  --launch-skip 1000 -c 1 -o "$out/sweep_cfg2" -f \
  python bench.py --steps 1100 --warmup 3 --no-cpu-baseline --no-extras \
  > "$out/ncu_full.log" 2>&1; echo "ncu full exit $?"
cat "$out/bench_cfg2.json"
