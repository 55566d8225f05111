#!/bin/bash
# row-walk order x grid size on the c2 probe (GPU box)
p() {
  echo "== fwd/SM=$1 grad/SM=$2 defines='$3'"
  SGB200_EW_DEFINES="$3" SGB200_EW_FWD_BLOCKS_PER_SM=$1 SGB200_EW_GRAD_BLOCKS_PER_SM=$2 \
    PYTHONPATH=. timeout -s KILL 120 python tools/ew_probe.py 2>&1 | head -1
}
B="#define SG_ROW_IL 0
#define SG_LD_CS 0"
p 64 8 "$B"
p 32 4 "$B"
p 96 6 "$B"
p 64 4 "$B
#define SG_GUNROLL 3"
p 64 8 "$B
#define SG_GUNROLL 3
#define SG_GRAD_MINB 3"
p 64 8 "$B
#define SG_UNROLL 2"
p 64 8 "$B
#define SG_ST_CS 0"
p 64 8 "$B"
