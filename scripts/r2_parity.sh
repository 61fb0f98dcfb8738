#!/usr/bin/env bash
# round-2 parity call: BASELINE-config oracle parity + the new window/warm-start tests
set -u
out=gpurun_out/r2b; mkdir -p $out
timeout 1500 python -m pytest tests/test_gpu_baseline_parity.py -m gpu -x -q -s --durations=0 > $out/baseline_parity.log 2>&1; echo "exit $?" >> $out/baseline_parity.log
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "window or wrong_size" > $out/small.log 2>&1; echo "exit $?" >> $out/small.log
tail -25 $out/baseline_parity.log; tail -3 $out/small.log
