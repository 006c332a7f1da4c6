bash tools/gpu/run_ncu.sh qs5 "k_apply_qs" apply3 4
bash tools/gpu/run_ncu.sh fdmcta8 "k_fdm_cta" fdm5
VARIANTS=0,4 timeout 600 python tools/time_apply.py --config config4 --p 4 2>&1 | grep "{"
