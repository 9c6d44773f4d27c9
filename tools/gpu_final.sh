# usage (under gpurun): bash tools/gpu_final.sh TAG -- the round's evidence: smoke, every gpu test,
# bench (C5), ncu launch list of the bench, ncu --set full of one k_heavy and one k_tiles launch
TAG=${1:-final}
mkdir -p gpurun_out
bash tools/gpu_full.sh $TAG
PSI_GRAPH=0 timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"^k_heavy$|^k_tiles$|^k_sell$" -s 4 -c 2 \
  -o gpurun_out/full_$TAG python tools/prof.py --config 5 > gpurun_out/ncu_full_$TAG.log 2>&1; echo ncu_full=$?
tail -2 gpurun_out/ncu_full_$TAG.log
