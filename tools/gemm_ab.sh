timeout 600 python -m pytest tests/test_gemm_gpu.py -q 2>&1 | tail -1
echo "== new"; timeout 300 python tools/prof_gemm.py 2>&1 | tail -9
echo "== v1"; TGB_GEMM_V1=1 timeout 300 python tools/prof_gemm.py 2>&1 | tail -9
timeout 300 python tools/bench_configs.py s2g 1,3 2>&1 | tail -2 | cut -c1-600
