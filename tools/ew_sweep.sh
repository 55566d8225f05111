#!/bin/bash
# Sweep fused-kernel tuning knobs on the c2 workload (run on the GPU box).
run() {
  echo "== defines='$1' fwd/SM=$2 grad/SM=$3"
  SGB200_EW_DEFINES="$1" SGB200_EW_FWD_BLOCKS_PER_SM=$2 SGB200_EW_GRAD_BLOCKS_PER_SM=$3 timeout -s KILL 300 \
    python bench.py --steps 20 --warmup 3 --no-cpu-baseline --secondary none 2>&1 | tail -1 |
    python -c "import json,sys; r=json.loads(sys.stdin.read()); print(r['value'], r['kernels_ms'])"
}
if [ $# -gt 0 ]; then run "$@"; exit; fi
run "" 4 8
run "#define SG_GUNROLL 4
#define SG_GRAD_MINB 2" 4 4
run "#define SG_GUNROLL 4
#define SG_GRAD_MINB 3" 4 6
run "#define SG_GRAD_MINB 3" 4 6
run "#define SG_GRAD_MINB 2" 4 4
run "#define SG_UNROLL 8" 2 8
run "#define SG_UNROLL 8" 4 8
run "#define SG_UNROLL 2" 8 8
