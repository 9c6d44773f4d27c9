# round 2 session 4, call c: k_sell with one load variant (PSI_EXP_SELL_ONELOAD) at C2 (sell forced, 64-row windows), C4, C5
mkdir -p gpurun_out
export PSI_SELL=1 PSI_SELL_SHIFT=6
CFG=2 bash tools/exp_build.sh none -DPSI_EXP_SELL_ONELOAD > gpurun_out/sell_oneload_c2.txt 2>&1
unset PSI_SELL PSI_SELL_SHIFT
CFG=4 bash tools/exp_build.sh none -DPSI_EXP_SELL_ONELOAD > gpurun_out/sell_oneload_c4.txt 2>&1
CFG=5 bash tools/exp_build.sh none -DPSI_EXP_SELL_ONELOAD none > gpurun_out/sell_oneload_c5.txt 2>&1
cat gpurun_out/sell_oneload_c*.txt
