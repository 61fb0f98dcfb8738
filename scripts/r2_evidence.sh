#!/usr/bin/env bash
# per-config evidence for BASELINE.md section 4: oracle parity numbers (-s), device
# rates of cfg 1/3/4/5 (bench lines), CPU reference arm on cfg 3 and 4
set -u
out=gpurun_out/${1:-r2e}; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_baseline_parity.py tests/test_gpu_parity.py -m gpu -q -s \
  -k "baseline or cfg or config1_full" > $out/parity.log 2>&1; echo "parity exit $?"
grep -E "^cfg|config1" $out/parity.log
for c in cfg1 cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > $out/bench_$c.json 2> $out/bench_$c.err
  echo "bench $c exit $?"
done
for c in cfg3 cfg4; do
  timeout 900 python bench.py --impl reference --config $c --steps 2 --warmup 1 > $out/ref_$c.json 2> $out/ref_$c.err
  echo "ref $c exit $?"
done
