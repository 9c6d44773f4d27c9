"""Wall-clock breakdown of the e2e path (the bench's e2e leg): psi_build_graph from pinned host
arrays, psi_iterate(eps), psi_get_psi to pinned host, destroy -- repeated.

    python tools/e2e_breakdown.py [--config 5] [--reps 4]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--reps", type=int, default=4)
    args = ap.parse_args()
    import numpy as np
    import torch
    import paper_2206_09960_b200 as psi
    sys.path.insert(0, ROOT)
    import bench
    w = bench.make_workload(args.config, seed=0, pinned=True)
    host = [torch.from_numpy(a) for a in (w.row_ptr, w.followers, w.lam, w.mu)]
    out = torch.empty(w.n, dtype=torch.float64, pin_memory=True)
    torch.cuda.synchronize()
    for r in range(args.reps):
        t0 = time.perf_counter()
        g = psi.PsiGraph(*host)
        t1 = time.perf_counter()
        g.iterate(w.eps)
        t2 = time.perf_counter()
        g.get_psi(out=out)
        t3 = time.perf_counter()
        info = g.info()
        g.close()
        torch.cuda.synchronize()
        t4 = time.perf_counter()
        print(f"rep {r}: build {1e3*(t1-t0):7.1f} ms (ingest kernels {info['ingest_ms']:7.1f})  "
              f"iterate {1e3*(t2-t1):6.1f}  get_psi {1e3*(t3-t2):6.1f}  destroy {1e3*(t4-t3):6.1f}  "
              f"total {1e3*(t4-t0):7.1f} ms", flush=True)


if __name__ == "__main__":
    main()
