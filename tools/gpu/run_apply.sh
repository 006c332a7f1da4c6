# split-quad apply: parity + timing; FP64 pipe microbench
cd tools/microbench && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_pipes fp64_pipes.cu && /tmp/fp64_pipes > ../../gpurun_out/fp64_pipes.txt 2>&1; cd ../..
cat gpurun_out/fp64_pipes.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "ragged or every_order" 2>&1 | tail -5
VARIANTS=0,3,4 timeout 600 python tools/time_apply.py --config config3 2>&1 | grep -v "^\[" | tee gpurun_out/apply_qs.jsonl
for p in 3 6; do VARIANTS=0,3,4 timeout 600 python tools/time_apply.py --config config4 --p $p 2>&1 | grep "{" | tee -a gpurun_out/apply_qs.jsonl; done
