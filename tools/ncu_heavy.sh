# usage (under gpurun): bash tools/ncu_heavy.sh TAG [prof.py args] -- ncu --set full of one
# k_heavy launch at C5 (direct launches: PSI_GRAPH=0), source-level
TAG=$1; shift
export PSI_GRAPH=0
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_heavy$" -s 2 -c 1 \
    -o gpurun_out/heavy_$TAG python tools/prof.py --config 5 "$@" > gpurun_out/ncu_heavy_$TAG.log 2>&1
echo ncu_rc=$?
tail -3 gpurun_out/ncu_heavy_$TAG.log
