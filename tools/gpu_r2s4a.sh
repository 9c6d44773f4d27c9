# round 2 session 4, call a: k_heavy scan skip A/B at C5 and C4; ncu of k_tiles at C2
mkdir -p gpurun_out
CFG=5 bash tools/exp_build.sh none -DPSI_EXP_FULLSCAN none > gpurun_out/scanskip_c5.txt 2>&1
CFG=4 bash tools/exp_build.sh none -DPSI_EXP_FULLSCAN > gpurun_out/scanskip_c4.txt 2>&1
python -c "from paper_2206_09960_b200 import _build; _build.build(force=True)"
bash tools/ncu_sweep.sh 2 c2_s4 --iters 4 > gpurun_out/ncu_c2.txt 2>&1
cat gpurun_out/scanskip_c5.txt gpurun_out/scanskip_c4.txt gpurun_out/ncu_c2.txt
