#!/bin/bash
# Round-2 final evidence in one GPU call (outputs in gpurun_out/prof_r02d/):
# tests + smoke, the default bench and the reference arm (no profiler), then
# the ncu launch lists of the bench's own command (c2 headline; c5 step) and
# --set full captures of K2 and the c5 dX GEMM.
set -u
O=gpurun_out/prof_r02d
mkdir -p $O
export PYTHONPATH=$PWD
timeout -s KILL 900 python -m pytest tests -m gpu -q > $O/gputest.log 2>&1; echo "pytest rc=$?" >> $O/gputest.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout -s KILL 900 python bench.py > $O/bench_full.json.log 2> $O/bench_full.err || echo "bench failed"
timeout -s KILL 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json.log 2>&1 || echo "reference arm failed"
NCU="timeout -s KILL 900 ncu --clock-control none"
$NCU --metrics gpu__time_duration.sum -c 400 --csv --log-file $O/launches_c2.csv \
  python bench.py --steps 2 --warmup 1 --secondary none --no-cpu-baseline > $O/ncu_c2.log 2>&1
$NCU --metrics gpu__time_duration.sum -k regex:'gemm|k_' -c 400 --csv --log-file $O/launches_c5.csv \
  python tools/mlp_probe.py 1024 16 32768 nograph > /dev/null 2>&1
$NCU --set full --import-source on -k regex:'sg_ew_grad' -s 2 -c 1 -o $O/c2_k2 -f \
  python bench.py --steps 3 --warmup 3 --secondary none --no-cpu-baseline > /dev/null 2>&1
$NCU --set full --import-source on -k regex:gemm_tc_pair -s 2 -c 1 -o $O/c5_dx -f python tools/gemm_one.py dx > /dev/null 2>&1
python tools/power_probe.py 1024 16 32768 4 > $O/power.log 2>&1
python tools/power_probe.py 4096 4 65536 4 >> $O/power.log 2>&1
ls -la $O
