#!/bin/bash
# Round-2 evidence in one GPU call (outputs in gpurun_out/prof_r02/):
#   bench (no profiler) + reference arm, ncu launch lists of the c2 and c5 steps,
#   --set full captures of K2 (the headline kernel), the c5 dX / fwd GEMMs and
#   the c3 bf16 GEMMs, and the gemm / chain timelines.
set -u
O=gpurun_out/prof_r02
mkdir -p $O
export PYTHONPATH=$PWD
NCU="timeout -s KILL 900 ncu --clock-control none"
B="timeout -s KILL 900 python bench.py"
$B --steps 20 --warmup 5 > $O/bench_full.json.log 2> $O/bench_full.err || echo "bench failed"
$B --impl reference --steps 20 --warmup 5 > $O/bench_reference.json.log 2>&1 || echo "reference arm failed"
$NCU --metrics gpu__time_duration.sum -c 40 --csv --log-file $O/launches_c2.csv \
  $B --steps 3 --warmup 3 --secondary none --no-cpu-baseline > /dev/null 2>&1
$NCU --metrics gpu__time_duration.sum -k regex:'gemm|k_|sg_' -c 400 --csv --log-file $O/launches_c5.csv \
  python tools/mlp_probe.py 1024 16 32768 nograph > /dev/null 2>&1
$NCU --set full --import-source on -k regex:'sg_ew_grad' -s 2 -c 1 -o $O/c2_k2 -f \
  $B --steps 3 --warmup 3 --secondary none --no-cpu-baseline > /dev/null 2>&1
for k in dx fwd dw; do
  $NCU --set full --import-source on -k regex:gemm_tc_pair -s 2 -c 1 -o $O/c5_$k -f python tools/gemm_one.py $k > /dev/null 2>&1
done
$NCU --set full -k regex:gemm_tc -s 6 -c 3 -o $O/c3_gemm -f python tools/gemm_one.py fwd 8192 4096 4096 > /dev/null 2>&1
ls -la $O
