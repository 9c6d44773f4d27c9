# round 2 session 4, call d: auto sliced-ELL + fused finish (C2), one-load tiles (C2/C3): tests + all configs
mkdir -p gpurun_out
bash tools/gpu_tests.sh s4d "sell or config2 or config3 or solver or pagerank or contract or kappa or heavy or determinism or smoke"
python tools/all_configs.py --out gpurun_out/all_configs_s4d.json > gpurun_out/all_configs_s4d.log 2>&1; echo allcfg=$?
tail -8 gpurun_out/all_configs_s4d.log
