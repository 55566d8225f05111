#!/bin/bash
# Packed fp32x2 epilogue math (default library) vs the scalar forms
# (libsgb200_scalar.so, built by: bash tools/build_variant.sh scalar -DSG_EPI_SCALAR_MATH=1)
export PYTHONPATH=$PWD
O=gpurun_out/math_ab
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/test.log 2>&1; echo "rc=$?" >> $O/test.log
for lib in libsgb200.so libsgb200_scalar.so libsgb200.so libsgb200_scalar.so; do
  echo "== $lib" >> $O/ab.log
  SGB200_LIB=$lib timeout 300 python tools/gemm_epi_probe.py 32768 1024 1024 >> $O/ab.log 2>&1
  SGB200_LIB=$lib timeout 300 python tools/mlp_probe.py 1024 16 32768 >> $O/ab.log 2>&1
  SGB200_LIB=$lib timeout 300 python tools/mlp_probe.py 1024 16 4096 >> $O/ab.log 2>&1
  SGB200_LIB=$lib timeout 300 python tools/power_probe.py 1024 16 32768 3 >> $O/ab.log 2>&1
done
