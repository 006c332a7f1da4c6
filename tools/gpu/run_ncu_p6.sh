bash tools/gpu/run_ncu.sh qs6 "k_apply_qs" apply config4p6 4
bash tools/gpu/run_ncu.sh warp6 "k_apply_warp" apply config4p6 0
