# usage (under gpurun): bash tools/tune_h8.sh -- heavy tests + heavy-path settings on C5/C4
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "heavy or long_rows or config1 or determin or pagerank" > gpurun_out/pytest_gpu_h8.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu_h8.log
timeout 1500 python tools/sweep_tune.py --config 5 \
  --set PSI_HEAVY_MIN=64,PSI_HEAVY_LABELS=1048576 \
  --set PSI_HEAVY_MIN=64,PSI_HEAVY_LABELS=2097152 \
  --set PSI_HEAVY_MIN=64,PSI_HEAVY_LABELS=524288 \
  --set PSI_HEAVY_MIN=32,PSI_HEAVY_LABELS=2097152 \
  --set PSI_HEAVY_MIN=128,PSI_HEAVY_LABELS=2097152 \
  > gpurun_out/tune_h8.txt 2>&1; echo tune=$?
timeout 900 python tools/sweep_tune.py --config 4 \
  --set PSI_HEAVY=0 \
  --set PSI_HEAVY=1,PSI_HEAVY_LABELS=1048576 \
  --set PSI_HEAVY=1,PSI_HEAVY_LABELS=524288 \
  >> gpurun_out/tune_h8.txt 2>&1; echo tune4=$?
cat gpurun_out/tune_h8.txt
