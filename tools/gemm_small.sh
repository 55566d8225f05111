# small Dense-layer GEMMs (the per-GPU shards of c5 / c4 at 8 GPUs): CTA pair vs 1-SM tile widths
for a in "1024 4096" "1024 8192" "4096 8192"; do
  for bn in 0 256 128 64; do
    echo "== FORCE_BN=$bn"; SGB200_GEMM_FORCE_BN=$bn PYTHONPATH=. timeout 120 python tools/cublas_c5.py $a
  done
done
