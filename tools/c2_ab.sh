#!/bin/bash
# same-box A/B on the c2 headline (bench.py, 200 steps): gradient kernel walking the row spans
# last-to-first (SG_GRAD_REV 1) vs first-to-last (the default)
for i in 1 2 3; do
  echo -n "rev:  "; SGB200_EW_DEFINES="#define SG_GRAD_REV 1" timeout 300 python bench.py --no-cpu-baseline --secondary none 2>/dev/null | python tools/bench_summary.py /dev/stdin | head -1
  echo -n "fwd:  "; timeout 300 python bench.py --no-cpu-baseline --secondary none 2>/dev/null | python tools/bench_summary.py /dev/stdin | head -1
done
