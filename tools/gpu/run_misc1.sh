timeout 600 python bench.py --sweep-one 3:dense_o1 --steps 2 --warmup 1 2>&1 | grep SWEEP | cut -c1-400
timeout 600 python bench.py --sweep-one 6:dense_o1 --steps 1 --warmup 1 2>&1 | grep SWEEP | python -c "import sys,json; d=json.loads(sys.stdin.read()[6:]); print(d.get('apply'))"
bash tools/gpu/run_ncu.sh fdmw6 "k_fdm_warp" fdm3
