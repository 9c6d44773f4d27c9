# usage (under gpurun): bash tools/gpu_ovl.sh TAG -- overlapped-sweep parity subset + C5 timing
TAG=${1:-ovl}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1; echo build=$?
PSI_OVERLAP=1 timeout 900 python -m pytest tests -m gpu -x -q -k "heavy or config5_small or config4_small or long_rows or deterministic or pagerank" > gpurun_out/pytest_ovl_$TAG.log 2>&1; echo pytest_ovl=$?
tail -5 gpurun_out/pytest_ovl_$TAG.log
timeout 900 python tools/sweep_tune.py --config 5 --set PSI_OVERLAP=0 --set PSI_OVERLAP=1 ${SETS} > gpurun_out/tune_$TAG.txt 2>&1; echo tune=$?
cat gpurun_out/tune_$TAG.txt
