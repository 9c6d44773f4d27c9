# usage (under gpurun): bash tools/tile_exp.sh TAG -- PSI_TILE variants: parity subset + timing
TAG=${1:-t}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1; echo build=$?
PSI_TILE=256 timeout 900 python -m pytest tests -m gpu -x -q -k "config1 or config4_small or config5_small or tile_boundary or long_rows or random_small" > gpurun_out/pytest_t256_$TAG.log 2>&1; echo pytest256=$?
tail -2 gpurun_out/pytest_t256_$TAG.log
for C in 5 3 4 2; do
timeout 900 python tools/sweep_tune.py --config $C --set PSI_TILE=0 --set PSI_TILE=256 ${SETS} 2>&1 | grep -v "^N=" ; done
