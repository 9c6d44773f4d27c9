"""Per-launch sweep timing for several library settings on one generated graph.

    python tools/sweep_tune.py --config 5 [--scale S] --set PSI_HOT_MB=0,PSI_L2_FETCH=0 --set ...
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
    ap.add_argument("--sweeps", type=int, default=20)
    ap.add_argument("--set", action="append", default=[])
    args = ap.parse_args()
    import torch
    import paper_2206_09960_b200 as psi
    import psigen
    t0 = time.time()
    w = psigen.make_config(args.config, scale=args.scale)
    print(f"N={w.n} M={w.m} gen {time.time() - t0:.1f}s", flush=True)
    dev = [torch.from_numpy(a).cuda() for a in (w.row_ptr, w.followers, w.lam, w.mu)]
    for s in args.set or [""]:
        for kv in filter(None, s.split(",")):
            k, v = kv.split("=")
            os.environ[k] = v
        with psi.PsiGraph(*dev) as g:
            g.time_sweep(3)
            hv, a, b = g.time_sweep(args.sweeps)
            st, T, gap = g.iterate(w.eps)
            inf = g.info()
        byt = 4 * w.m + 4 * (w.n + 1) + 8 * inf["n_g"] + 32 * inf["n_f"]
        print(f"[{s}] k_heavy {hv:.3f} ms  k_tiles {a:.3f} ms  k_fix {b:.3f} ms  sweep {hv + a + b:.3f} ms  "
              f"{byt / (hv + a + b) / 1e6:.0f} GB/s  T={T} solve {inf['iterate_ms']:.2f} ms  "
              f"heavy rows {inf['n_heavy']} entries {inf['heavy_entries']} panels {inf['heavy_panels']}  "
              f"ingest {inf['ingest_ms']:.0f} ms", flush=True)


if __name__ == "__main__":
    main()
