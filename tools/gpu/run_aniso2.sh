timeout 1500 python -m pytest tests/test_gpu_aniso.py tests/test_gpu_fdm.py -m gpu -x -q 2>&1 | tail -3
