nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 3000 python -m pytest tests -m gpu -x -q --durations=30 > gpurun_out/r2s_gputests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r2s_gputests.log
timeout 900 python bench.py --no-sweep > gpurun_out/r2s_bench.json 2> gpurun_out/r2s_bench.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/r2s_bench.json
