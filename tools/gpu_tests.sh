# usage (under gpurun): bash tools/gpu_tests.sh TAG [pytest -k expr] [extra pytest args]
TAG=${1:-t}; K=${2:-}; shift 2; EXTRA="$@"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo smoke=$?
tail -2 gpurun_out/smoke_$TAG.log
if [ -n "$K" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -k "$K" $EXTRA > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest=$?
else
  timeout 1500 python -m pytest tests -m gpu -x -q $EXTRA > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest=$?
fi
tail -15 gpurun_out/pytest_gpu_$TAG.log
