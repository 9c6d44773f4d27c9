# round 2 session 5, call f: panel shape search, finer grid + tapered tail; trace shows the chosen shape
mkdir -p gpurun_out
bash tools/gpu_tests.sh s5h "small_scale or checked or heavy or config4"
for C in 4 5; do
PSI_TRACE=1 python tools/sweep_tune.py --config $C --set "" --set PSI_HEAVY_SEARCH=0 > gpurun_out/tune_heavy_search_c${C}_s5h.txt 2>&1
grep -v "^\[psi ingest\] [a-z +]" gpurun_out/tune_heavy_search_c${C}_s5h.txt | grep -E "panel shape|k_heavy"
done
