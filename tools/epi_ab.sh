#!/bin/bash
# A/B of the GEMM epilogue store paths on the c5 / c3 shapes (tools only):
# TMA bulk stores (default) vs direct stores, TMA-staged aux vs global loads.
export PYTHONPATH=$PWD
O=gpurun_out/epi_ab
mkdir -p $O
for v in "" "SGB200_GEMM_TMA_STORE=0" "SGB200_GEMM_AUX_TMA=0" "SGB200_GEMM_WIDE=1"; do
  for shape in "32768 1024 1024" "8192 4096 4096"; do
    echo "[$v] $shape" >> $O/epi.log
    env $v timeout 300 python tools/gemm_epi_probe.py $shape >> $O/epi.log 2>&1
  done
done
