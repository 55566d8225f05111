#!/bin/bash
# grid shape sweep on the c2 probe (GPU box): blocks per SM and block width (columns)
p() {
  echo "== fwd/SM=$1 fwdBDX=$2 grad/SM=$3 gradBDX=$4 defines='$5'"
  SGB200_EW_DEFINES="$5" SGB200_EW_FWD_BLOCKS_PER_SM=$1 SGB200_EW_FWD_BDX=$2 SGB200_EW_GRAD_BLOCKS_PER_SM=$3 \
    SGB200_EW_GRAD_BDX=$4 PYTHONPATH=. timeout -s KILL 120 python tools/ew_probe.py 2>&1 | head -1
}
p 64 256 8 256
p 128 256 8 64
p 256 256 8 32
p 64 64 32 64
p 128 128 16 128
p 32 256 32 32
p 64 256 64 16
p 64 256 8 64 "#define SG_LD_CS 0"
