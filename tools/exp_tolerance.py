"""Experiments 1-2 of the paper on synthetic stand-ins, written as CSV (SPEC S:386
format) -- the data behind DESIGN.md §11's Exp. 1/2 table.

    python tools/exp_tolerance.py [--out profiles/r1/exp12]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/exp12")
    args = ap.parse_args()
    import numpy as np
    import torch
    import paper_2206_09960_b200 as psi
    from paper_2206_09960_b200 import experiments
    import psigen
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    n, m, seed = 12_591, 49_743, 0            # DBLP's size (Table II)
    rp, f = psigen.chung_lu_graph(n, m, 2.1, 400.0, seed)   # power-law stand-in
    cases = {
        "heterogeneous": (psigen.uniform(n, 1e-6, 1.0, seed, 1), psigen.uniform(n, 1e-6, 1.0, seed, 2),
                          ("power_psi", "power_nf"), None),
        "homogeneous": (np.full(n, 0.15), np.full(n, 0.85), ("power_psi", "power_nf", "pagerank"), 0.85),
    }
    for name, (lam, mu, methods, alpha) in cases.items():
        dev = [torch.from_numpy(a).cuda() for a in (rp, f, lam, mu)]
        with psi.PsiGraph(*dev) as g:
            rows, _ = experiments.tolerance_sweep(g, methods=methods, alpha=alpha)
        with psi.PsiGraph(*dev) as g:
            g.iterate(1e-14)
            ref = g.get_psi().cpu().numpy()
            curves = {mm: experiments.error_curve(g, mm, range(0, 160, 4) if mm != "power_nf" else range(0, 60, 6),
                                                  alpha=alpha, reference=ref) for mm in methods}
        cpath = f"{args.out}_{name}_curves.csv"
        with open(cpath, "w") as fh:
            fh.write(f"# Fig. 4-5 style: matvecs vs Eq. (23) error, {name} activity, fixed-count runs\n")
            fh.write("method,t,matvecs,error\n")
            for mm, cv in curves.items():
                for t, mv, err in cv:
                    fh.write(f"{mm},{t},{mv},{err:.6e}\n")
        hdr = (f"Exp. 1/2 (P:414-433), {name} activity, Chung-Lu (gamma 2.1) stand-in for DBLP: N={n}, M={f.size}, seed {seed}\n"
               f"reference: Power-psi at eps=1e-14 on the GPU; error = Eq. (23); B200, {torch.cuda.get_device_name()}")
        path = f"{args.out}_{name}.csv"
        open(path, "w").write(experiments.to_csv(rows, hdr))
        print(open(path).read())


if __name__ == "__main__":
    main()
