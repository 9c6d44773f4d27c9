TAG=${1:-r1c}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
B="PSI_GROUPS=1,PSI_SMEM_HOT=0"
timeout 1500 python tools/sweep_tune.py --config 5 \
  --set $B,PSI_HOT_MB=42,PSI_L1_HOT=4096 \
  --set $B,PSI_HOT_MB=42,PSI_L1_HOT=8192 \
  --set $B,PSI_HOT_MB=42,PSI_L1_HOT=16384 \
  --set $B,PSI_HOT_MB=42,PSI_L1_HOT=32768 \
  --set $B,PSI_HOT_MB=42,PSI_L1_HOT=262144 \
  --set $B,PSI_HOT_MB=42,PSI_L1_HOT=2000000000 \
  --set $B,PSI_HOT_MB=64,PSI_L1_HOT=16384 \
  --set $B,PSI_HOT_MB=80,PSI_L1_HOT=16384 \
  --set $B,PSI_HOT_MB=32,PSI_L1_HOT=16384 \
  --set PSI_GROUPS=2,PSI_SMEM_HOT=0,PSI_HOT_MB=42,PSI_L1_HOT=16384 \
  --set PSI_GROUPS=4,PSI_SMEM_HOT=0,PSI_HOT_MB=42,PSI_L1_HOT=16384 \
  --set PSI_GROUPS=4,PSI_SMEM_HOT=4096,PSI_HOT_MB=42,PSI_L1_HOT=16384 \
  > gpurun_out/tune_$TAG.txt 2>&1; echo tune=$?
timeout 900 python tools/sweep_tune.py --config 4 \
  --set $B,PSI_HOT_MB=42,PSI_L1_HOT=0 \
  --set $B,PSI_HOT_MB=42,PSI_L1_HOT=16384 \
  --set $B,PSI_HOT_MB=42,PSI_L1_HOT=2000000000 \
  >> gpurun_out/tune_$TAG.txt 2>&1; echo tune4=$?
cat gpurun_out/tune_$TAG.txt
