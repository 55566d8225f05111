#!/bin/bash
# same-box A/B of the gradient-kernel configuration on the c2 headline (bench.py, 200 steps)
OLD="SGB200_EW_GRAD_BLOCKS_PER_SM=8"
OLDDEF="#define SG_GRAD_MINB 4
#define SG_GUNROLL 3"
for i in 1 2 3; do
  echo -n "new: "; timeout 300 python bench.py --no-cpu-baseline --secondary none 2>/dev/null | python tools/bench_summary.py /dev/stdin | head -1
  echo -n "old: "; env $OLD SGB200_EW_DEFINES="$OLDDEF" timeout 300 python bench.py --no-cpu-baseline --secondary none 2>/dev/null | python tools/bench_summary.py /dev/stdin | head -1
done
