#!/usr/bin/env bash
# round-2 final evidence in one call: the whole GPU suite (with the printed parity numbers),
# smoke, the driver's two bench arms, bench lines of configs 1/3/4/5 and the ALCC arm, the
# launch list of the default bench command and one full ncu capture of its sweep.
#   gpurun --timeout 3000 -- 'bash scripts/r2_final.sh r2l'
set -u
tag=${1:-r2l}; out=gpurun_out/$tag; mkdir -p $out
(nproc; free -g | head -2; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv) > $out/host.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -s --durations=12 > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" | tee -a $out/pytest_gpu.log
grep -E "vs compiled|live reference|GPU vs reference|^cfg|passed|failed" $out/pytest_gpu.log | tail -24
python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke exit $?"; tail -2 $out/smoke.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $out/ref.json 2> $out/ref.err; echo "ref exit $?"
timeout 900 python bench.py --steps 20 --warmup 5 > $out/bench.json 2> $out/bench.err; echo "bench exit $?"
for c in cfg1 cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > $out/bench_$c.json 2> $out/bench_$c.err
  echo "bench $c exit $?"
done
timeout 600 python bench.py --solver alcc --steps 20 --warmup 5 --no-cpu-baseline > $out/bench_alcc.json 2> $out/bench_alcc.err; echo "alcc exit $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extras > $out/ncu_launch.log 2>&1; echo "launch list exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_mma_kernel --launch-skip 12 -c 1 \
  -o $out/sweep_cfg2_it13 -f python bench.py --steps 17 --warmup 3 --no-cpu-baseline --no-extras > $out/ncu_full.log 2>&1; echo "ncu full exit $?"
python - <<PY
import json
def last(p):
    return json.loads(open(p).read().strip().splitlines()[-1])
d = last('$out/bench.json'); r = d['roofline']
print('cfg2 value', d['value'] / 1e9, 'ms', d['ms_per_step'], 'frac', r['frac'], 'model24', r['model_24B_per_pair_frac'],
      'share', r['sweep_share_of_step'], 'e2e', d['e2e']['value'] / 1e9, 'launches', d['gpu_launches'])
print('ttt', json.dumps(d.get('time_to_tolerance')))
print('cpu', json.dumps(d.get('cpu_baseline')))
print('port', json.dumps(d.get('cpu_port_allcores')), json.dumps(d.get('cpu_baseline_1thread')))
print('other', json.dumps(d.get('other_configs')))
print('clocks', json.dumps(d.get('clocks')))
f = last('$out/ref.json'); print('ref', f['value'] / 1e9, f['cpu_baseline']['kind'], f.get('cpu_port_allcores', {}).get('value'))
for c in ('cfg1', 'cfg3', 'cfg4', 'cfg5', 'alcc'):
    try:
        b = last('$out/bench_%s.json' % c); print(c, b['value'] / 1e9, b['ms_per_step'], b['roofline']['frac'], b.get('clocks', {}).get('reasons'))
    except Exception as e:
        print(c, 'failed', e)
PY
