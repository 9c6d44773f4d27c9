# round 2 session 5, call j: staged labels H and the heavy-row threshold re-tuned with the panel shape search (C4, C5)
mkdir -p gpurun_out
python tools/sweep_tune.py --config 4 --set "" --set PSI_HEAVY_LABELS=786432 --set PSI_HEAVY_LABELS=1048576 \
  --set PSI_HEAVY_LABELS=524288,PSI_HEAVY_MIN=48 --set PSI_HEAVY_LABELS=524288,PSI_HEAVY_MIN=96 \
  --set PSI_HEAVY_LABELS=786432,PSI_HEAVY_MIN=48 > gpurun_out/tune_heavy_h_c4_s5j.txt 2>&1
cat gpurun_out/tune_heavy_h_c4_s5j.txt
python tools/sweep_tune.py --config 5 --set "" --set PSI_HEAVY_MIN=48 --set PSI_HEAVY_MIN=96 \
  --set PSI_HEAVY_LABELS=786432,PSI_HEAVY_MIN=64 > gpurun_out/tune_heavy_h_c5_s5j.txt 2>&1
cat gpurun_out/tune_heavy_h_c5_s5j.txt
python tools/sweep_tune.py --config 3 --set "" --set PSI_HEAVY=1,PSI_HEAVY_LABELS=65536 --set PSI_HEAVY=1,PSI_HEAVY_LABELS=131072 \
  --set PSI_HEAVY=1,PSI_HEAVY_LABELS=262144 --set PSI_HEAVY=1,PSI_HEAVY_LABELS=524288 \
  --set PSI_HEAVY=1,PSI_HEAVY_LABELS=131072,PSI_HEAVY_MIN=128 --set PSI_HEAVY=1,PSI_HEAVY_LABELS=131072,PSI_SELL=0 \
  > gpurun_out/tune_heavy_h_c3_s5j.txt 2>&1
cat gpurun_out/tune_heavy_h_c3_s5j.txt
