# round 2 session 5, call a: k_heavy_balance permuting every portion of a run inside its block (long runs too)
mkdir -p gpurun_out
bash tools/gpu_tests.sh s5a "small_scale or checked or heavy or config4"
python tools/sweep_tune.py --config 5 > gpurun_out/tune_c5_s5a.txt 2>&1
python tools/sweep_tune.py --config 4 > gpurun_out/tune_c4_s5a.txt 2>&1
cat gpurun_out/tune_c5_s5a.txt gpurun_out/tune_c4_s5a.txt
bash tools/ncu_heavy.sh s5a
