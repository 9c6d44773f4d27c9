# usage (under gpurun): bash tools/gpu_base.sh TAG  -- build + C5 per-launch sweep timing (defaults)
TAG=${1:-base}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1; echo build=$?
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_$TAG.txt
timeout 900 python tools/sweep_tune.py --config 5 ${SETS} > gpurun_out/tune_$TAG.txt 2>&1; echo tune=$?
cat gpurun_out/tune_$TAG.txt
