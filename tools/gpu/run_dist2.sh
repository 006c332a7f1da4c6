timeout 1200 python -m pytest tests/test_gpu_dist.py -m gpu -x -q 2>&1 | tail -2
for ov in 0 1; do
  echo "== SEM_DIST_OVERLAP=$ov"
  SEM_DIST_OVERLAP=$ov timeout 600 python bench.py --smoother fdm --emulate-ranks 4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-variants --no-sweep 2>/dev/null | tail -1 | cut -c1-300
done
