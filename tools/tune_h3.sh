TAG=${1:-h3}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 1500 python tools/sweep_tune.py --config 5 \
  --set PSI_HEAVY=0 \
  --set PSI_HEAVY=1,PSI_HEAVY_MIN=128,PSI_HEAVY_SEGS=128 \
  --set PSI_HEAVY=1,PSI_HEAVY_MIN=64,PSI_HEAVY_SEGS=128 \
  --set PSI_HEAVY=1,PSI_HEAVY_MIN=32,PSI_HEAVY_SEGS=128 \
  --set PSI_HEAVY=1,PSI_HEAVY_MIN=64,PSI_HEAVY_SEGS=256 \
  --set PSI_HEAVY=1,PSI_HEAVY_MIN=64,PSI_HEAVY_SEGS=512 \
  --set PSI_HEAVY=1,PSI_HEAVY_MIN=256,PSI_HEAVY_SEGS=256 \
  > gpurun_out/tune_$TAG.txt 2>&1; echo tune=$?
timeout 900 python tools/sweep_tune.py --config 4 \
  --set PSI_HEAVY=0 \
  --set PSI_HEAVY=1,PSI_HEAVY_MIN=128,PSI_HEAVY_SEGS=128 \
  --set PSI_HEAVY=1,PSI_HEAVY_MIN=64,PSI_HEAVY_SEGS=128 \
  --set PSI_HEAVY=1,PSI_HEAVY_MIN=64,PSI_HEAVY_SEGS=256 \
  >> gpurun_out/tune_$TAG.txt 2>&1; echo tune4=$?
cat gpurun_out/tune_$TAG.txt
