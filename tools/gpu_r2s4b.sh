# round 2 session 4, call b: sliced-ELL window size and one-load gathers at C2 / C3
mkdir -p gpurun_out
python -c "from paper_2206_09960_b200 import _build; _build.build(force=True)"
for C in 2 3; do
python tools/sweep_tune.py --config $C --set "" --set PSI_SELL=1,PSI_SELL_SHIFT=5 --set PSI_SELL_SHIFT=6 \
  --set PSI_SELL_SHIFT=7 --set PSI_SELL_SHIFT=6,PSI_SELL_KCAP=64 --set PSI_SELL_SHIFT=6,PSI_SELL_KCAP=32 \
  --set PSI_SELL=0,PSI_SMEM_HOT=0 --set PSI_SMEM_HOT=0,PSI_L1_HOT=0 > gpurun_out/sell_small_c$C.txt 2>&1
done
CFG=2 bash tools/exp_build.sh none -DPSI_EXP_ONELOAD=1 -DPSI_EXP_ONELOAD=2 > gpurun_out/oneload_c2.txt 2>&1
CFG=3 bash tools/exp_build.sh none -DPSI_EXP_ONELOAD=1 -DPSI_EXP_ONELOAD=2 > gpurun_out/oneload_c3.txt 2>&1
cat gpurun_out/sell_small_c2.txt gpurun_out/sell_small_c3.txt gpurun_out/oneload_c2.txt gpurun_out/oneload_c3.txt
