TAG=${1:-c1}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "heavy or long_rows or config1 or config4 or determin or random" > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 1500 python tools/sweep_tune.py --config 5 \
  --set PSI_CONCURRENT=1 \
  --set PSI_CONCURRENT=0 \
  --set PSI_CONCURRENT=1,PSI_HEAVY_MIN=128 \
  --set PSI_CONCURRENT=1,PSI_HEAVY_MIN=64,PSI_HEAVY_SEGS=512 \
  --set PSI_CONCURRENT=1,PSI_HEAVY_MIN=64,PSI_HEAVY_SEGS=128 \
  --set PSI_CONCURRENT=1,PSI_HEAVY_MIN=64,PSI_HEAVY_SEGS=256,PSI_SMEM_HOT=0 \
  > gpurun_out/tune_$TAG.txt 2>&1; echo tune=$?
timeout 900 python tools/sweep_tune.py --config 4 \
  --set PSI_HEAVY=0 \
  --set PSI_HEAVY=1,PSI_CONCURRENT=1,PSI_HEAVY_SEGS=128 \
  --set PSI_HEAVY=1,PSI_CONCURRENT=1,PSI_HEAVY_SEGS=256 \
  >> gpurun_out/tune_$TAG.txt 2>&1; echo tune4=$?
cat gpurun_out/tune_$TAG.txt
