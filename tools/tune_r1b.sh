# usage (under gpurun): bash tools/tune_r1b.sh TAG
TAG=${1:-r1b}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu_$TAG.log
S="PSI_HOT_MB=42,PSI_L1_HOT=0"
timeout 1500 python tools/sweep_tune.py --config 5 \
  --set PSI_GROUPS=1,PSI_SMEM_HOT=0,$S \
  --set PSI_GROUPS=4,PSI_SMEM_HOT=0,$S \
  --set PSI_GROUPS=4,PSI_SMEM_HOT=16384,$S \
  --set PSI_GROUPS=4,PSI_SMEM_HOT=20000,$S \
  --set PSI_GROUPS=2,PSI_SMEM_HOT=24000,$S \
  --set PSI_GROUPS=2,PSI_SMEM_HOT=12000,$S \
  --set PSI_GROUPS=1,PSI_SMEM_HOT=0,PSI_HOT_MB=42,PSI_L1_HOT=16384 \
  --set PSI_GROUPS=1,PSI_SMEM_HOT=0,PSI_HOT_MB=42,PSI_L1_HOT=65536 \
  --set PSI_GROUPS=4,PSI_SMEM_HOT=16384,PSI_HOT_MB=42,PSI_L1_HOT=24576 \
  --set PSI_GROUPS=4,PSI_SMEM_HOT=16384,PSI_HOT_MB=0,PSI_L1_HOT=0 \
  --set PSI_GROUPS=4,PSI_SMEM_HOT=16384,PSI_HOT_MB=24,PSI_L1_HOT=0 \
  --set PSI_GROUPS=4,PSI_SMEM_HOT=16384,PSI_HOT_MB=56,PSI_L1_HOT=0 \
  > gpurun_out/tune_$TAG.txt 2>&1; echo tune=$?
cat gpurun_out/tune_$TAG.txt
