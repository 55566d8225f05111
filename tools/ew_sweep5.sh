#!/bin/bash
# ROW-partial accumulator placement (registers vs shared memory) on the c2 probe
p() {
  echo "== grad/SM=$1 defines='$2'"
  SGB200_EW_DEFINES="$2" SGB200_EW_GRAD_BLOCKS_PER_SM=$1 PYTHONPATH=. timeout -s KILL 120 python tools/ew_probe.py 2>&1 | grep -E "affsig|R,1|1-elem"
}
p 8 ""
p 8 "#define SG_ROW_SMEM 1
#define SG_GUNROLL 3"
p 7 "#define SG_ROW_SMEM 1
#define SG_GUNROLL 3"
p 8 "#define SG_ROW_SMEM 1
#define SG_GUNROLL 3"
