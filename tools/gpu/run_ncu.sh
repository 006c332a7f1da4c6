# usage: bash tools/gpu/run_ncu.sh <tag> <kernel-regex> <ncu_target args...>
# one ncu --set full capture (source-level) of the first matching launch; report + source CSV to gpurun_out/
tag=$1; kre=$2; shift 2
python tools/ncu_target.py "$@" > gpurun_out/ncu_${tag}_plain.log 2>&1 || { echo "plain run failed"; tail gpurun_out/ncu_${tag}_plain.log; exit 1; }
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"$kre" -c 1 -f -o gpurun_out/ncu_${tag} \
  python tools/ncu_target.py "$@" > gpurun_out/ncu_${tag}.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/ncu_${tag}.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ncu_${tag}_source.csv 2>/dev/null
ncu -i gpurun_out/ncu_${tag}.ncu-rep --page raw --csv > gpurun_out/ncu_${tag}_raw.csv 2>/dev/null
ls -la gpurun_out/ncu_${tag}*
