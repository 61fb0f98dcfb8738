#!/usr/bin/env bash
# round-2 full call: GPU tests, the default driver bench line (CPU legs included), reference arm
set -u
tag=${1:-r2f}; tests=${2:-all}
out=gpurun_out/$tag; mkdir -p $out
(nproc; free -g | head -2) > $out/host.txt 2>&1
if [ "$tests" = all ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > $out/pytest_gpu.log 2>&1; echo "exit $?" >> $out/pytest_gpu.log
  tail -22 $out/pytest_gpu.log
fi
timeout 900 python bench.py --steps 20 --warmup 5 > $out/bench.json 2> $out/bench.err; echo bench $?
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $out/ref.json 2> $out/ref.err; echo ref $?
python - <<PY
import json
d=json.loads(open('$out/bench.json').read().strip().splitlines()[-1]); r=d['roofline']
print('value',d['value']/1e9,'ms',d['ms_per_step'],'frac',r['frac'],'share',r['sweep_share_of_step'],'e2e',d['e2e']['value']/1e9)
print('ttt',json.dumps(d.get('time_to_tolerance')))
print('cpu',json.dumps(d.get('cpu_baseline')),json.dumps(d.get('cpu_baseline_1thread')))
print('other',json.dumps(d.get('other_configs')))
f=json.loads(open('$out/ref.json').read().strip().splitlines()[-1]); print('ref',f['value']/1e9, f.get('steps'), f.get('warmup'), f['cpu_baseline']['sample'])
PY
