#!/bin/bash
# gradient kernel: register budget (SG_GRAD_MINB blocks/SM) x rows in flight x grid
p() {
  echo "== grad/SM=$1 defines='$2'"
  SGB200_EW_DEFINES="$2" SGB200_EW_GRAD_BLOCKS_PER_SM=$1 PYTHONPATH=. timeout -s KILL 120 python tools/ew_probe.py 2>&1 | grep -E "affsig|R,1|1-elem|f64"
}
p 8 ""
for minb in 3 2; do
  for u in 4 5 6 8; do
    for bps in 3 6; do
      p $((bps * minb / 3)) "#define SG_GRAD_MINB $minb
#define SG_GUNROLL $u"
    done
  done
done
