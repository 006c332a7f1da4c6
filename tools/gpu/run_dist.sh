timeout 1200 python -m pytest tests/test_gpu_dist.py -m gpu -x -q 2>&1 | tail -2
SEM_DIST_OVERLAP=0 SEM_DIST_GRAPHS=0 timeout 1200 python -m pytest tests/test_gpu_dist.py -m gpu -x -q 2>&1 | tail -2
for g in 0 1; do
  echo "== SEM_DIST_GRAPHS=$g"
  SEM_DIST_GRAPHS=$g timeout 600 python bench.py --emulate-ranks 4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-variants --no-sweep 2>/dev/null | tail -1 | cut -c1-400
  SEM_DIST_GRAPHS=$g timeout 600 python bench.py --config config2 --emulate-ranks 4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-variants --no-sweep 2>/dev/null | tail -1 | cut -c1-400
done
bash tools/gpu/run_ncu.sh qs5b "k_apply_qs" apply3 4
