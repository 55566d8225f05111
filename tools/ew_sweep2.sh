#!/bin/bash
# load/store cache-hint and grid-size sweep on the c2 probe (GPU box)
p() {
  echo "== defines='$1' fwd/SM=$2 grad/SM=$3"
  SGB200_EW_DEFINES="$1" SGB200_EW_FWD_BLOCKS_PER_SM=$2 SGB200_EW_GRAD_BLOCKS_PER_SM=$3 PYTHONPATH=. \
    timeout -s KILL 120 python tools/ew_probe.py 2>&1 | head -2
}
p "" 4 8
p "#define SG_LD_CS 0" 4 8
p "#define SG_ST_CS 0" 4 8
p "#define SG_LD_CS 0
#define SG_ST_CS 0" 4 8
p "" 16 8
p "" 64 8
p "#define SG_LD_CS 0
#define SG_ST_CS 0" 64 8
