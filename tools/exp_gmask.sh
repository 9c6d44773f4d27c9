# usage (under gpurun): bash tools/exp_gmask.sh -- the edge-stream kernel with x gathers confined to 2^k labels
# (experiment builds: results are wrong by construction; only the sweep time is of interest)
mkdir -p gpurun_out
cat > /tmp/ts.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
import paper_2206_09960_b200 as psi, psigen
w = psigen.make_config(5)
dev = [torch.from_numpy(a).cuda() for a in (w.row_ptr, w.followers, w.lam, w.mu)]
with psi.PsiGraph(*dev) as g:
    g.time_sweep(3)
    print(sys.argv[1], "k_heavy %.3f k_sell|k_tiles %.3f k_fix %.3f" % g.time_sweep(20), flush=True)
PY
for M in none 0x3FFFFF 0x7FFFFF 0xFFFFFF; do
  if [ $M = none ]; then export PSI_NVCC_EXTRA=""; else export PSI_NVCC_EXTRA="-DPSI_EXP_GMASK=$M"; fi
  python -c "from paper_2206_09960_b200 import _build; _build.build(force=True)" || exit 1
  timeout 600 python /tmp/ts.py $M
done
