# A/B of the branch-uniform FDM kernels (v5) against the previous build (libsem_pmg_v4.so), the
# tests that reach the FDM kernels, then the default bench
V=$PWD/paper_2009_00705_b200/libsem_pmg_v4.so
for c in config5 config3; do
  SEM_PMG_LIB=$V CONFIG=$c python tools/time_fdm.py > gpurun_out/ab5_fdm_${c}_v4.txt 2>&1
  CONFIG=$c python tools/time_fdm.py > gpurun_out/ab5_fdm_${c}_v5.txt 2>&1
done
grep -h "fdm sweep" gpurun_out/ab5_fdm_*
python -m pytest tests/test_gpu_fdm.py tests/test_gpu_dist.py tests/test_gpu_det.py tests/test_gpu_fnpf.py tests/test_gpu_nextstage.py tests/test_gpu_condense.py tests/test_gpu_aniso.py -m gpu -x -q > gpurun_out/ab5_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/ab5_tests.log
timeout 1200 python bench.py > gpurun_out/r2v_bench_default.json 2> gpurun_out/r2v_bench_default.err; echo "bench rc=$?"
tail -c 300 gpurun_out/r2v_bench_default.json
