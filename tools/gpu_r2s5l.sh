# round 2 session 5, call l: plan default first, search + second pass only when worth it; warm-build host plan wait
mkdir -p gpurun_out
bash tools/gpu_tests.sh s5l "small_scale or checked or heavy or config4"
for C in 4 5; do
PSI_TRACE=1 python tools/sweep_tune.py --config $C --set PSI_HEAVY_SEARCH=0 --set PSI_HEAVY_SEARCH=1 --set PSI_HEAVY_SEARCH=1 > gpurun_out/tune_heavy_search_c${C}_s5l.txt 2>&1
grep -E "panel shape|k_heavy|host plan joined" gpurun_out/tune_heavy_search_c${C}_s5l.txt
done
