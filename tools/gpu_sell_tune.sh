# usage (under gpurun): SETS="--set ..." bash tools/gpu_sell_tune.sh TAG -- k_sell settings at C3/C5,
# then ncu --set full of one k_sell launch (C3 and C5, library defaults + PSI_SELL=1)
TAG=${1:-st}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1; echo build=$?
for C in ${CONFIGS:-3 5}; do
  timeout 900 python tools/sweep_tune.py --config $C $SETS > gpurun_out/tune_${TAG}_c$C.txt 2>&1; echo tune_c$C=$?
  cat gpurun_out/tune_${TAG}_c$C.txt
done
if [ "${NCU:-1}" = "1" ]; then
for C in ${NCU_CONFIGS:-3 5}; do
  PSI_SELL=1 PSI_GRAPH=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_sell$" -s 1 -c 1 \
    -o gpurun_out/sell_${TAG}_c$C python tools/prof.py --config $C > gpurun_out/ncu_sell_${TAG}_c$C.log 2>&1; echo ncu_c$C=$?
done
fi
