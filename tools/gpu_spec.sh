timeout 900 python -m pytest tests/test_spectrum_gpu.py tests/test_reduction_gpu.py -x -q -m gpu 2>&1 | tail -15
