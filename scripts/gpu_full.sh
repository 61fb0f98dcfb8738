#!/usr/bin/env bash
# End-of-milestone evidence in one gpurun call: GPU tests, bench lines for the
# five BASELINE configs, the reference arm, ALCC and general-K arms, the cfg 2
# launch list and `ncu --set full` sweep captures (cfg 2 at iteration ~1000,
# cfg 3 at ~300).  gpurun --timeout 3600 -- 'bash scripts/gpu_full.sh <tag>'
set -u
tag=${1:-r}
out=gpurun_out/$tag
mkdir -p "$out"
timeout 1200 python -m pytest tests -m gpu -x -q > "$out/pytest_gpu.log" 2>&1; echo "pytest exit $?" >> "$out/pytest_gpu.log"
tail -2 "$out/pytest_gpu.log"
timeout 600 python bench.py > "$out/bench_cfg2.json" 2> "$out/bench_cfg2.err"
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > "$out/bench_reference.json" 2> "$out/bench_reference.err"
for c in cfg1 cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --config $c --steps 200 > "$out/bench_$c.json" 2> "$out/bench_$c.err"
done
timeout 600 python bench.py --solver alcc --steps 300 > "$out/bench_alcc.json" 2> "$out/bench_alcc.err"
timeout 600 python bench.py --solver papg-alcc --config cfg1 --steps 5 > "$out/bench_general_k2.json" 2> "$out/bench_general_k2.err"
timeout 600 python bench.py --solver papg-alcc --config cfg1 --K 40 --steps 5 > "$out/bench_general_k40.json" 2> "$out/bench_general_k40.err"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file "$out/launches.csv" python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extras \
  > "$out/ncu_launch.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_mma_kernel \
  --launch-skip 1000 -c 1 -o "$out/sweep_cfg2" -f \
  python bench.py --steps 1100 --warmup 3 --no-cpu-baseline --no-extras > "$out/ncu_full.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_mma_kernel \
  --launch-skip 300 -c 1 -o "$out/sweep_cfg3" -f \
  python bench.py --config cfg3 --steps 400 --warmup 3 --no-cpu-baseline --no-extras > "$out/ncu_full3.log" 2>&1
for f in "$out"/bench_*.json; do echo "$f: $(head -c 300 "$f")"; done
