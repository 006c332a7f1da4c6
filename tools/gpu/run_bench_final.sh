timeout 3000 python bench.py > gpurun_out/r2s_bench_final2.json 2> gpurun_out/r2s_bench_final2.err; echo "bench rc=$?"
tail -c 600 gpurun_out/r2s_bench_final2.json
