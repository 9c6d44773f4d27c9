TAG=${1:-r1e}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python tools/sweep_tune.py --config 5 \
  --set PSI_ST_LAST=1,PSI_SINGLE_L1=0,PSI_HOT_MB=42 \
  --set PSI_ST_LAST=0,PSI_SINGLE_L1=0,PSI_HOT_MB=42 \
  --set PSI_ST_LAST=0,PSI_SINGLE_L1=1,PSI_HOT_MB=42 \
  --set PSI_ST_LAST=0,PSI_SINGLE_L1=1,PSI_HOT_MB=32 \
  --set PSI_ST_LAST=0,PSI_SINGLE_L1=1,PSI_HOT_MB=56 \
  --set PSI_ST_LAST=0,PSI_SINGLE_L1=1,PSI_HOT_MB=64 \
  --set PSI_ST_LAST=0,PSI_SINGLE_L1=1,PSI_HOT_MB=72 \
  --set PSI_ST_LAST=0,PSI_SINGLE_L1=1,PSI_HOT_MB=90 \
  > gpurun_out/tune_$TAG.txt 2>&1; echo tune=$?
timeout 900 python tools/sweep_tune.py --config 4 \
  --set PSI_ST_LAST=1,PSI_SINGLE_L1=0,PSI_HOT_MB=42 \
  --set PSI_ST_LAST=0,PSI_SINGLE_L1=1,PSI_HOT_MB=42 \
  --set PSI_ST_LAST=0,PSI_SINGLE_L1=1,PSI_HOT_MB=64 \
  >> gpurun_out/tune_$TAG.txt 2>&1; echo tune4=$?
cat gpurun_out/tune_$TAG.txt
