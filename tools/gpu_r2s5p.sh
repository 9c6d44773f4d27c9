# round 2 session 5, call p: panel search thresholds at C5 (gate / gain knobs); k_sell without loads for padding (-DPSI_EXP_SENT)
mkdir -p gpurun_out
PSI_TRACE=1 python tools/sweep_tune.py --config 5 --set "" --set PSI_HEAVY_SEARCH_GATE=0,PSI_HEAVY_SEARCH_GAIN=2 \
  --set PSI_HEAVY_SEARCH_GATE=0,PSI_HEAVY_SEARCH_GAIN=0 > gpurun_out/tune_heavy_gain_c5_s5p.txt 2>&1
grep -E "panel shape|k_heavy" gpurun_out/tune_heavy_gain_c5_s5p.txt
CFG=5 bash tools/exp_build.sh none "-DPSI_EXP_SENT" > gpurun_out/exp_sent_c5_s5p.txt 2>&1
CFG=4 bash tools/exp_build.sh "-DPSI_EXP_SENT" none > gpurun_out/exp_sent_c4_s5p.txt 2>&1
CFG=2 bash tools/exp_build.sh none "-DPSI_EXP_SENT" > gpurun_out/exp_sent_c2_s5p.txt 2>&1
cat gpurun_out/exp_sent_c?_s5p.txt
