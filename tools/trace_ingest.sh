# usage (under gpurun): bash tools/trace_ingest.sh CONFIG [--set ...] -- ingest phase times + sweep time
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
CFG=${1:-5}; shift
PSI_TRACE=1 timeout 900 python tools/sweep_tune.py --config $CFG "$@" > gpurun_out/trace_ingest.log 2>&1
cat gpurun_out/trace_ingest.log
