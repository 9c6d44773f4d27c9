# round 2 session 5, call d: panel shape search (simulated claim order) at C4 / C5 / forced-heavy C3
mkdir -p gpurun_out
bash tools/gpu_tests.sh s5d "small_scale or checked or heavy or config4"
for C in 4 5; do
python tools/sweep_tune.py --config $C --set "" --set PSI_HEAVY_SEARCH=0 > gpurun_out/tune_heavy_search_c${C}_s5d.txt 2>&1
cat gpurun_out/tune_heavy_search_c${C}_s5d.txt
done
