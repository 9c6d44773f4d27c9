# round 2 session 5, call k: new heavy-plan knob tests; C2 k_sell occupancy / hot-cache sweep
mkdir -p gpurun_out
bash tools/gpu_tests.sh s5k "heavy_rows_parity"
python tools/sweep_tune.py --config 2 --set "" --set PSI_SMEM_HOT=0 --set PSI_SMEM_HOT=0,PSI_L1_HOT=0 > gpurun_out/tune_c2_a_s5k.txt 2>&1
python tools/sweep_tune.py --config 2 --set PSI_SELL_WARPS=24 > gpurun_out/tune_c2_b_s5k.txt 2>&1
python tools/sweep_tune.py --config 2 --set PSI_SELL_WARPS=16 > gpurun_out/tune_c2_c_s5k.txt 2>&1
python tools/sweep_tune.py --config 2 --set PSI_SELL_KCAP=512,PSI_SELL_SHIFT=7 > gpurun_out/tune_c2_d_s5k.txt 2>&1
cat gpurun_out/tune_c2_?_s5k.txt
