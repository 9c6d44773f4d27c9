"""Small end-to-end exercise of every kernel (ingest, k_heavy, k_tiles, k_fix, readout,
PageRank, unpermute) for compute-sanitizer:

    compute-sanitizer --tool memcheck python tools/sanitize_small.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2206_09960_b200 as psi
    import psigen
    os.environ["PSI_HEAVY"] = "1"
    os.environ["PSI_HEAVY_MIN"] = "8"
    for cfg, scale, ovl in ((1, None, "0"), (5, 15, "0"), (3, 14, "0"), (5, 15, "1")):
        os.environ["PSI_OVERLAP"] = ovl         # the overlapped plan's kernels too (last pass)
        w = psigen.make_config(cfg, scale=scale)
        dev = [torch.from_numpy(a).cuda() for a in (w.row_ptr, w.followers, w.lam, w.mu)]
        with psi.PsiGraph(*dev) as g:
            g.iterate(w.eps)
            p = g.get_psi().cpu()
            g.get_series()
            g.pagerank(0.85, 1e-9)
            g.get_pagerank()
            g.time_sweep(2)
            g.iterate(0.0, 3)
            if w.m <= 1 << 27:
                g.power_nf([0, 1, w.n - 1], 1e-9)
            info = g.info()
        with psi.PsiGraph(w.row_ptr, w.followers, w.lam, w.mu) as g:   # host inputs
            g.iterate(w.eps)
        print(f"config {cfg}: n={w.n} m={w.m} heavy={info['n_heavy']} overlapped={info['overlapped']} "
              f"sum(psi)={float(p.sum()):.12f}",
              flush=True)


if __name__ == "__main__":
    main()
