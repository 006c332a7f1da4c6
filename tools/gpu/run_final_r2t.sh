# end-of-session evidence (round 2, session 4): full GPU tests, default bench, launch lists of the
# headline step (config 3) and config 5, one ncu --set full capture of k_fdm_cta<8>
python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/r2u_gputests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2u_gputests.log
timeout 1500 python bench.py > gpurun_out/r2u_bench_default.json 2> gpurun_out/r2u_bench_default.err; echo "bench rc=$?"
SEM_NO_GRAPHS=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/r2u_launches_config3.csv python tools/profile_step.py --config config3 > gpurun_out/r2u_prof3.log 2>&1; echo "ncu3 rc=$?"
SEM_NO_GRAPHS=1 timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/r2u_launches_config5.csv python tools/profile_step.py --config config5 --smoother fdm > gpurun_out/r2u_prof5.log 2>&1; echo "ncu5 rc=$?"
bash tools/gpu/run_ncu.sh r2u_fdm_cta8 "k_fdm_cta" fdm5
python tools/ncu_source_top.py gpurun_out/ncu_r2u_fdm_cta8_source.csv 40 > gpurun_out/r2u_fdm_cta8_source_top.txt
tail -c 400 gpurun_out/r2u_bench_default.json
