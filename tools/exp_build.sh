# usage (under gpurun): bash tools/exp_build.sh "FLAGS1" "FLAGS2" ... -- C5 sweep timing per
# experiment build (PSI_NVCC_EXTRA; "none" = the product build)
mkdir -p gpurun_out
cat > /tmp/ts.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
import paper_2206_09960_b200 as psi, psigen
w = psigen.make_config(int(sys.argv[2]) if len(sys.argv) > 2 else 5)
dev = [torch.from_numpy(a).cuda() for a in (w.row_ptr, w.followers, w.lam, w.mu)]
with psi.PsiGraph(*dev) as g:
    g.time_sweep(3)
    print(sys.argv[1], "k_heavy %.3f k_tiles %.3f k_fix %.3f" % g.time_sweep(20), flush=True)
PY
for F in "$@"; do
  if [ "$F" = none ]; then export PSI_NVCC_EXTRA=""; else export PSI_NVCC_EXTRA="$F"; fi
  python -c "from paper_2206_09960_b200 import _build; _build.build(force=True)" || exit 1
  timeout 600 python /tmp/ts.py "$F" ${CFG:-5}
done
