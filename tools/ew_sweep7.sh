#!/bin/bash
# gradient kernel after the per-group fp32 pre-sums: rows in flight x grid size
p() {
  echo "== grad/SM=$1 defines='$2'"
  SGB200_EW_DEFINES="$2" SGB200_EW_GRAD_BLOCKS_PER_SM=$1 PYTHONPATH=. timeout -s KILL 120 python tools/ew_probe.py 2>&1 | grep -E "affsig|R,1|1-elem"
}
for bps in 4 8 16; do
  p $bps "#define SG_GUNROLL 2"
  p $bps "#define SG_GUNROLL 3"
done
p 8 "#define SG_GUNROLL 2
#define SG_ROW_SMEM 0"
p 16 "#define SG_GUNROLL 2
#define SG_ROW_SMEM 0"
p 8 "#define SG_GUNROLL 4"
