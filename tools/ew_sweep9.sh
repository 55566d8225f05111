#!/bin/bash
# forward kernel: register budget (SG_FWD_MINB) x rows in flight x grid size
p() {
  echo "== fwd/SM=$1 defines='$2'"
  SGB200_EW_DEFINES="$2" SGB200_EW_FWD_BLOCKS_PER_SM=$1 PYTHONPATH=. timeout -s KILL 120 python tools/ew_probe.py 2>&1 | grep -E "affsig"
}
p 64 ""
for mb in 5 6 8; do
  for u in 2 3 4; do
    p 64 "#define SG_FWD_MINB $mb
#define SG_UNROLL $u"
  done
done
