timeout 1200 python -m pytest tests/test_gpu_aniso.py tests/test_gpu_parity.py -m gpu -x -q -k "aniso or ragged or every_order or Aniso or level" 2>&1 | tail -2
for lib in ab/libsem_pmg_r2d.so paper_2009_00705_b200/libsem_pmg.so; do
  echo "== $lib"
  SEM_PMG_LIB=$PWD/$lib timeout 900 python tools/time_apply_aniso.py 2>&1 | grep "{"
done
