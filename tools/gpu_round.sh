# usage (under gpurun): bash tools/gpu_round.sh TAG
# build -> smoke -> pytest -m gpu -> bench (C5) -> ncu launch list of bench -> ncu --set full of k_tiles
TAG=${1:-r1}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/nvsmi_$TAG.txt
free -g >> gpurun_out/nvsmi_$TAG.txt; nproc >> gpurun_out/nvsmi_$TAG.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu_$TAG.log
timeout 1200 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench=$?
cat gpurun_out/bench_$TAG.json
if [ "${SKIP_NCU:-0}" = "0" ]; then
PSI_GRAPH=0 timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu \
  > gpurun_out/ncu_launch_$TAG.log 2>&1; echo ncu_launch=$?
PSI_GRAPH=0 timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_tiles -s 4 -c 1 \
  -o gpurun_out/full_$TAG python tools/prof.py --config 5 > gpurun_out/ncu_full_$TAG.log 2>&1; echo ncu_full=$?
fi
