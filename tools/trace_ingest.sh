# usage (under gpurun): bash tools/trace_ingest.sh CONFIG -- ingest phase times + sweep time, twice
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
PSI_TRACE=1 timeout 900 python tools/sweep_tune.py --config ${1:-5} --set PSI_TRACE=1 --set PSI_TRACE=1 > gpurun_out/trace_ingest.log 2>&1
cat gpurun_out/trace_ingest.log
