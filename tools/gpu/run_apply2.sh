timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "ragged or every_order" 2>&1 | tail -3
VARIANTS=0,4 timeout 600 python tools/time_apply.py --config config3 2>&1 | grep "{"
for p in 3 4 6; do VARIANTS=4 timeout 600 python tools/time_apply.py --config config4 --p $p 2>&1 | grep "{"; done
