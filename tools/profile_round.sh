#!/bin/bash
# One GPU call: bench without a profiler first, then the ncu launch lists and
# --set full captures of the top kernels (outputs in gpurun_out/prof_$TAG).
set -u
TAG=${1:-r02}
O=gpurun_out/prof_$TAG
mkdir -p $O
NCU="ncu --clock-control none"
B="timeout -s KILL 600 python bench.py --no-cpu-baseline"
$B --steps 10 --warmup 3 --secondary c3,c5 > $O/bench.log 2>&1 || { echo "bench failed"; tail -20 $O/bench.log; exit 1; }
tail -c 600 $O/bench.log
# launch lists (per-launch durations, cold cache, serialised)
$NCU --metrics gpu__time_duration.sum -k regex:'sg_ew_|k_sum' -c 24 --csv --log-file $O/launches_c2.csv \
  $B --steps 3 --warmup 3 --secondary none > /dev/null 2>&1
$NCU --metrics gpu__time_duration.sum -k regex:'gemm|k_act|k_colsum|k_splitk' -c 40 --csv --log-file $O/launches_c3.csv \
  $B --steps 3 --warmup 3 --rows 1024 --secondary c3 > /dev/null 2>&1
$NCU --metrics gpu__time_duration.sum -k regex:'gemm|k_act|k_colsum|k_splitk|k_mse|k_sgd|k_sum_loss' -c 300 --csv \
  --log-file $O/launches_c5.csv $B --steps 3 --warmup 3 --rows 1024 --secondary c5 > /dev/null 2>&1
# full sections of the top kernels
$NCU --set full --import-source on -k regex:'sg_ew_' -s 4 -c 2 -o $O/c2_ew -f \
  $B --steps 3 --warmup 3 --secondary none > /dev/null 2>&1
$NCU --set full --import-source on -k regex:'gemm_tc' -c 3 -o $O/c3_gemm -f \
  $B --steps 1 --warmup 3 --rows 1024 --secondary c3 > /dev/null 2>&1
ls -la $O
