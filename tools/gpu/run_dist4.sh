timeout 1200 python -m pytest tests/test_gpu_dist.py tests/test_gpu_nccl.py -m gpu -x -q 2>&1 | tail -2
timeout 600 python bench.py --smoother fdm --emulate-ranks 4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-variants --no-sweep 2>/dev/null | tail -1 | cut -c1-200
timeout 600 python bench.py --emulate-ranks 4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-variants --no-sweep 2>/dev/null | tail -1 | cut -c1-200
# final round-2 evidence: launch lists of the headline step (config 3) and config 5, then the full default bench
SEM_NO_GRAPHS=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/r2s_launches_config3.csv python tools/profile_step.py --config config3 > gpurun_out/r2s_prof3.log 2>&1; echo "ncu3 rc=$?"
SEM_NO_GRAPHS=1 timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/r2s_launches_config5.csv python tools/profile_step.py --config config5 --smoother fdm > gpurun_out/r2s_prof5.log 2>&1; echo "ncu5 rc=$?"
timeout 3000 python bench.py > gpurun_out/r2s_bench_final.json 2> gpurun_out/r2s_bench_final.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/r2s_bench_final.json
