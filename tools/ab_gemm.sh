# DGEMM rasterisation A/B: TGB_GEMM_GROUP=0 (column-major grid) vs 8 (grouped)
for G in 0 8; do echo "== group $G"; TGB_GEMM_GROUP=$G timeout 300 python tools/prof_gemm.py 2>&1 | tail -10
  TGB_GEMM_GROUP=$G timeout 300 python tools/bench_configs.py g$G 1 2>&1 | grep -o '"coulomb_ms": [0-9.]*\|"reduce_rank_ms": [0-9.]*\|"density_tensor_device_ms": [0-9.]*'
done
