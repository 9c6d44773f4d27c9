# usage (under gpurun): bash tools/gpu_quick.sh TAG [pytest -k expr]
TAG=${1:-q}; K=${2:-}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo smoke=$?
tail -2 gpurun_out/smoke_$TAG.log
if [ -n "$K" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest=$?
else
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest=$?
fi
tail -15 gpurun_out/pytest_gpu_$TAG.log
