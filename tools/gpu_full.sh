# usage (under gpurun): bash tools/gpu_full.sh TAG -- smoke, all gpu tests, bench C5, launch list
TAG=${1:-full}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/nvsmi_$TAG.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo smoke=$?
tail -1 gpurun_out/smoke_$TAG.log
timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest=$?
tail -22 gpurun_out/pytest_gpu_$TAG.log
timeout 1200 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench=$?
cat gpurun_out/bench_$TAG.json
if [ "${NCU:-1}" = "1" ]; then
PSI_GRAPH=0 timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-batch --no-configs \
  > gpurun_out/ncu_launch_$TAG.log 2>&1; echo ncu_launch=$?
fi
