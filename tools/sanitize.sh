#!/bin/bash
# compute-sanitizer over tools/sanitize_cases.py (one GPU call); summaries in gpurun_out/sanitize/.
set -u
O=gpurun_out/sanitize
mkdir -p $O
export PYTHONPATH=$PWD
CS="timeout -s KILL 900 compute-sanitizer --print-limit 20 --error-exitcode 9"
for tool in memcheck synccheck racecheck; do
  for c in fused gemm1 pair splitk tail actgrad small chain step loss; do
    $CS --tool $tool python tools/sanitize_cases.py $c > $O/${tool}_$c.log 2>&1
    echo "$tool $c rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|Error' $O/${tool}_$c.log | tail -1)"
  done
done | tee $O/summary.txt
