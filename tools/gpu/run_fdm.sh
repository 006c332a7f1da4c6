timeout 1200 python -m pytest tests/test_gpu_fdm.py -m gpu -x -q 2>&1 | tail -3
CONFIG=config5 timeout 900 python tools/time_fdm.py 2>&1 | grep "level"
timeout 600 python tools/time_fdm.py 2>&1 | grep "level"
