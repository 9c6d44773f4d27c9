"""Small driver for ncu: ingest one config and run a few fixed-count solves.

    python tools/prof.py --config 5 [--scale S] [--iters 3] [--solves 2]
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
    ap.add_argument("--scale", type=int, default=None)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--solves", type=int, default=2)
    ap.add_argument("--eps", type=float, default=0.0)
    ap.add_argument("--batch", type=int, default=0, help="k activity profiles (batch context)")
    args = ap.parse_args()
    import torch
    import paper_2206_09960_b200 as psi
    import psigen
    t0 = time.time()
    w = psigen.make_config(args.config, scale=args.scale)
    print(f"generated N={w.n} M={w.m} in {time.time() - t0:.1f}s", flush=True)
    lam, mu = w.lam, w.mu
    if args.batch > 1:
        lam, mu = psigen.activity_profiles(w.n, args.batch, "lognormal")
    dev = [torch.from_numpy(a).cuda() for a in (w.row_ptr, w.followers, lam, mu)]
    with psi.PsiGraph(*dev) as g:
        for _ in range(args.solves):
            if args.batch > 1:          # direct launches (graph kernel nodes are not profiled)
                print("batch sweep ms", g.time_sweep_batch(args.iters))
            st, T, gap = g.iterate(args.eps, args.iters)
        info = g.info()
    print(f"T={T} gap={gap:.3e} iterate_ms={info['iterate_ms']:.3f} ingest_ms={info['ingest_ms']:.1f}"
          f" tiles={info['num_tiles']} split={info['num_long_rows']} grid={info['grid']}")


if __name__ == "__main__":
    main()
