TAG=${1:-ph}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
export PSI_GRAPH=0
python tools/prof.py --config 5 > gpurun_out/prof_plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"^k_heavy$|k_tiles" -s 4 -c 2 \
    -o gpurun_out/full_$TAG python tools/prof.py --config 5 > gpurun_out/ncu_full_$TAG.log 2>&1
echo ncu=$?
