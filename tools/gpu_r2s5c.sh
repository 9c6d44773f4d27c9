# round 2 session 5, call c: k_heavy plan shape (segment size x slots per panel) at C5 and C4
mkdir -p gpurun_out
for C in 5 4; do
python tools/sweep_tune.py --config $C --set "" --set PSI_HEAVY_SEG_SHIFT=12,PSI_HEAVY_SLOTS=16384 \
  --set PSI_HEAVY_SEG_SHIFT=12,PSI_HEAVY_SLOTS=12288 --set PSI_HEAVY_SEG_SHIFT=12,PSI_HEAVY_SLOTS=8192 \
  --set PSI_HEAVY_SEG_SHIFT=13,PSI_HEAVY_SLOTS=10240 --set PSI_HEAVY_SEG_SHIFT=13,PSI_HEAVY_SLOTS=6144 \
  --set PSI_HEAVY_SEG_SHIFT=12,PSI_HEAVY_SLOTS=16384,PSI_HEAVY_LABELS=1572864 \
  --set PSI_HEAVY_SEG_SHIFT=12,PSI_HEAVY_SLOTS=16384,PSI_HEAVY_LABELS=1048576,PSI_HEAVY_MIN=48 \
  > gpurun_out/tune_heavy_shape_c${C}_s5c.txt 2>&1
cat gpurun_out/tune_heavy_shape_c${C}_s5c.txt
done
