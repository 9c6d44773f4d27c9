"""e2e variance diagnosis: repeated build (pinned host inputs) / iterate / get / destroy at a
config with PSI_TRACE=1, so every build prints its ingest phases (host and device time).

    PSI_TRACE=1 python tools/e2e_trace.py [--config 5] [--reps 8]
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
    ap.add_argument("--reps", type=int, default=8)
    a = ap.parse_args()
    import torch
    import paper_2206_09960_b200 as psi
    import bench
    w = bench.make_workload(a.config, seed=0, pinned=True)
    host = [torch.from_numpy(x) for x in (w.row_ptr, w.followers, w.lam, w.mu)]
    out = torch.empty(w.n, dtype=torch.float64, pin_memory=True)
    torch.cuda.synchronize()
    for r in range(a.reps):
        t0 = time.perf_counter()
        g = psi.PsiGraph(*host)
        t1 = time.perf_counter()
        g.iterate(w.eps)
        g.get_psi(out=out)
        t2 = time.perf_counter()
        info = g.info()
        g.close()
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        print(f"rep {r}: build {1e3*(t1-t0):7.1f} (device {info['ingest_ms']:.1f})  iterate+get "
              f"{1e3*(t2-t1):6.1f}  destroy {1e3*(t3-t2):6.1f} ms", file=sys.stderr, flush=True)


if __name__ == "__main__":
    main()
