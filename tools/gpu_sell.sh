# usage (under gpurun): bash tools/gpu_sell.sh TAG -- sliced-ELL sweep: its parity tests, then
# per-launch sweep times against the tiles at C3 / C4 / C5
TAG=${1:-sell}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_sell.py -x -q > gpurun_out/pytest_sell_$TAG.log 2>&1; echo pytest_sell=$?
tail -5 gpurun_out/pytest_sell_$TAG.log
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_$TAG.txt
for C in ${CONFIGS:-3 5}; do
  timeout 900 python tools/sweep_tune.py --config $C --set PSI_SELL=0 --set PSI_SELL=1 ${SETS} > gpurun_out/tune_${TAG}_c$C.txt 2>&1; echo tune_c$C=$?
  cat gpurun_out/tune_${TAG}_c$C.txt
done
