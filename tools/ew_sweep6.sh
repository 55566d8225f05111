#!/bin/bash
# forward kernel: rows in flight x grid size on the c2 probe
p() {
  echo "== fwd/SM=$1 defines='$2'"
  SGB200_EW_DEFINES="$2" SGB200_EW_FWD_BLOCKS_PER_SM=$1 PYTHONPATH=. timeout -s KILL 120 python tools/ew_probe.py 2>&1 | head -1
}
p 64 ""
p 64 "#define SG_UNROLL 8"
p 32 "#define SG_UNROLL 8"
p 128 "#define SG_UNROLL 2"
p 96 ""
p 64 "#define SG_UNROLL 6"
