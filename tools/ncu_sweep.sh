# usage (under gpurun): bash tools/ncu_sweep.sh <config> <tag> [extra prof.py args]
# Direct stream launches (PSI_GRAPH=0): ncu cannot profile kernel nodes of conditional graphs.
export PSI_GRAPH=0
CFG=$1; TAG=$2; shift 2
python tools/prof.py --config $CFG "$@" > gpurun_out/prof_plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python tools/prof.py --config $CFG "$@" > gpurun_out/ncu_launch_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_tiles -s 2 -c 1 \
    -o gpurun_out/prof_$TAG python tools/prof.py --config $CFG "$@" > gpurun_out/ncu_full_$TAG.log 2>&1
echo ncu_rc=$?
tail -3 gpurun_out/prof_plain_$TAG.log
