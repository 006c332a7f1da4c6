timeout 900 python -m pytest tests/test_gpu_fdm.py -m gpu -x -q 2>&1 | tail -2
for lib in ab/libsem_pmg_r2d.so paper_2009_00705_b200/libsem_pmg.so; do
  echo "== $lib"
  SEM_PMG_LIB=$PWD/$lib CONFIG=config5 timeout 900 python tools/time_fdm.py 2>&1 | grep "^level"
  SEM_PMG_LIB=$PWD/$lib timeout 900 python tools/time_fdm.py 2>&1 | grep "^level"
done
