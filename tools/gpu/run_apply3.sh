timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "ragged or every_order" 2>&1 | tail -2
for lib in ab/libsem_pmg_base.so ab/libsem_pmg_stager.so paper_2009_00705_b200/libsem_pmg.so; do
  echo "== $lib"
  SEM_PMG_LIB=$PWD/$lib VARIANTS=0 timeout 600 python tools/time_apply.py --config config3 2>&1 | grep "{" | cut -c1-200
  SEM_PMG_LIB=$PWD/$lib VARIANTS=0 timeout 600 python tools/time_apply.py --config config4 --p 3 2>&1 | grep "{" | cut -c1-200
done
