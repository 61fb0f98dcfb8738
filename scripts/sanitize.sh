#!/usr/bin/env bash
# compute-sanitizer memcheck / racecheck / synccheck over the sanitize_cases.py solves
set -u
out=gpurun_out/${1:-r2san}; mkdir -p $out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for c in sweep small fused sigma sigma_grid alcc general; do
    timeout 600 $CS --tool $tool --error-exitcode 9 --print-limit 20 python scripts/sanitize_cases.py $c \
      > $out/${tool}_${c}.log 2>&1
    echo "$tool $c exit $? : $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|error' $out/${tool}_${c}.log | tail -1)"
  done
done
