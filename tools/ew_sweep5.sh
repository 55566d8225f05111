#!/bin/bash
p() {
  echo "== grad/SM=$1 defines='$2'"
  SGB200_EW_DEFINES="$2" SGB200_EW_GRAD_BLOCKS_PER_SM=$1 PYTHONPATH=. timeout -s KILL 120 python tools/ew_probe.py 2>&1 | head -2
}
p 8 "#define SG_ACC_ROWS 1"
p 8 ""
p 8 "#define SG_ACC_ROWS 16"
p 8 "#define SG_ACC_ROWS 4"
p 12 ""
p 8 "#define SG_GUNROLL 4
#define SG_GRAD_MINB 3"
