# round 2 session 4, call e: fused k_sell finish with 16 loads in flight; C3 shared-memory hot copy sizes (one-load tiles)
mkdir -p gpurun_out
bash tools/gpu_tests.sh s4e "sell_fused or config2"
python tools/sweep_tune.py --config 2 > gpurun_out/tune_c2_s4e.txt 2>&1
python tools/sweep_tune.py --config 3 --set "" --set PSI_SMEM_HOT=8192 --set PSI_SMEM_HOT=12288 --set PSI_SMEM_HOT=16384 \
  --set PSI_SMEM_HOT=20480 --set PSI_SMEM_HOT=2048 > gpurun_out/tune_c3_smemhot_s4e.txt 2>&1
cat gpurun_out/tune_c2_s4e.txt gpurun_out/tune_c3_smemhot_s4e.txt
