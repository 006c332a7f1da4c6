timeout 3000 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/r2s_gputests_final.log 2>&1; echo "tests rc=$?"
tail -22 gpurun_out/r2s_gputests_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
