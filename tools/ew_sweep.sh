#!/bin/bash
# Tuning sweeps of the fused broadcast kernels on the c2 probe (GPU box).
#
#   tools/ew_sweep.sh one FWD_BPS GRAD_BPS 'DEFINES'   one configuration
#   tools/ew_sweep.sh grad                              K2: register budget x rows in flight x grid
#   tools/ew_sweep.sh fwd                               K1: register budget x rows in flight x grid
#   tools/ew_sweep.sh rowacc                            K2: ROW partials in registers vs shared memory
#
# Knobs: SGB200_EW_FWD_BLOCKS_PER_SM / SGB200_EW_GRAD_BLOCKS_PER_SM (grid size)
# and SGB200_EW_DEFINES (#defines prepended to the NVRTC source: SG_UNROLL,
# SG_GUNROLL, SG_FWD_MINB, SG_GRAD_MINB, SG_ROW_SMEM, SG_ROW_IL, SG_LD_CS, SG_ST_CS).
# (Replaces round 1's ew_sweep.sh, ew_sweep4..9.sh.)
export PYTHONPATH=.
p() {  # fwd/SM grad/SM defines [grep pattern]
  echo "== fwd/SM=$1 grad/SM=$2 defines='$3'"
  SGB200_EW_DEFINES="$3" SGB200_EW_FWD_BLOCKS_PER_SM=$1 SGB200_EW_GRAD_BLOCKS_PER_SM=$2 \
    timeout -s KILL 120 python tools/ew_probe.py 2>&1 | grep -E "${4:-affsig|R,1|1-elem|f64}"
}
case "${1:-grad}" in
  one) p "$2" "$3" "$4" ;;
  grad)
    p 64 8 ""
    for minb in 3 2; do
      for u in 4 5 6 8; do
        for bps in 3 6; do
          p 64 $((bps * minb / 3)) "#define SG_GRAD_MINB $minb
#define SG_GUNROLL $u"
        done
      done
    done ;;
  fwd)
    p 64 8 "" affsig
    for mb in 5 6 8; do
      for u in 2 3 4; do
        p 64 8 "#define SG_FWD_MINB $mb
#define SG_UNROLL $u" affsig
      done
    done ;;
  rowacc)
    for bps in 4 8 16; do
      p 64 $bps "#define SG_GUNROLL 2
#define SG_ROW_SMEM 0"
      p 64 $bps "#define SG_GUNROLL 2
#define SG_ROW_SMEM 1"
    done ;;
esac
