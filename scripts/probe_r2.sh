set -u
out=gpurun_out/r2a; mkdir -p $out
(nproc; lscpu | head -20; free -g; cat /proc/meminfo | head -3; nvidia-smi) > $out/host.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu.log
tail -3 $out/pytest_gpu.log
timeout 300 python bench.py --steps 20 --warmup 5 > $out/bench.json 2> $out/bench.err; echo bench $?
cat $out/bench.json | head -c 600
