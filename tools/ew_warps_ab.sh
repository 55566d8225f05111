#!/bin/bash
# A/B of the CTA-pair kernel's epilogue warp count (SGB200_GEMM_EW=8|12|16):
# parity first (GEMM + Dense tests under each), then GEMM and step timings.
export PYTHONPATH=$PWD
O=gpurun_out/ew_warps
mkdir -p $O
for ew in 12 16; do
  SGB200_GEMM_EW=$ew timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_dense_gpu.py tests/test_baseline_sizes_gpu.py -q -x > $O/test_$ew.log 2>&1
  echo "rc=$?" >> $O/test_$ew.log
done
for ew in 8 12 16; do
  for shape in "32768 1024 1024" "8192 4096 4096" "4096 1024 1024"; do
    echo "EW=$ew $shape" >> $O/epi.log
    SGB200_GEMM_EW=$ew timeout 300 python tools/gemm_epi_probe.py $shape >> $O/epi.log 2>&1
  done
done
for ew in 8 12 16 8; do
  for cfg in "1024 16 32768" "1024 16 4096" "4096 4 65536"; do
    echo "EW=$ew" >> $O/mlp.log; SGB200_GEMM_EW=$ew timeout 300 python tools/mlp_probe.py $cfg >> $O/mlp.log 2>&1
  done
done
