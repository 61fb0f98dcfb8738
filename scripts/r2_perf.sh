#!/usr/bin/env bash
# round-2 iteration call: GPU tests (optional), per-phase sweep timing at cfg 2, short bench
set -u
tag=${1:-r2c}; tests=${2:-tests}
out=gpurun_out/$tag; mkdir -p $out
if [ "$tests" = tests ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "exit $?" >> $out/pytest_gpu.log
  tail -3 $out/pytest_gpu.log
fi
timeout 300 python scripts/phase_perf.py 10000 10 > $out/phase.txt 2>&1; cat $out/phase.txt
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $out/bench.json 2> $out/bench.err; echo bench $?
python -c "
import json;d=json.loads(open('$out/bench.json').read().strip().splitlines()[-1]);print('value',d['value']/1e9,'ms',d['ms_per_step'],'frac',d['roofline']['frac'],'e2e',d['e2e']['value']/1e9, 'ttt', d.get('time_to_tolerance',{}).get('seconds'))"
