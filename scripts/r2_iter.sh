#!/usr/bin/env bash
# iteration call: sweep parity tests, per-launch sweep times (stream vs isolated), short bench
set -u
tag=${1:-r2i}; tests=${2:-parity}
out=gpurun_out/$tag; mkdir -p $out
if [ "$tests" = parity ]; then
  timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > $out/pytest_parity.log 2>&1; echo "exit $?" >> $out/pytest_parity.log
  tail -3 $out/pytest_parity.log
elif [ "$tests" = all ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "exit $?" >> $out/pytest_gpu.log
  tail -3 $out/pytest_gpu.log
fi
timeout 300 python scripts/stream_vs_isolated.py 25 > $out/svi.txt 2>&1; grep "step mean" $out/svi.txt
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extras > $out/bench.json 2> $out/bench.err; echo bench $?
python -c "
import json;d=json.loads(open('$out/bench.json').read().strip().splitlines()[-1]);r=d['roofline'];print('value',d['value']/1e9,'ms',d['ms_per_step'],'frac',r['frac'],'share',r['sweep_share_of_step'])"
