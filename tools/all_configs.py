"""GTEPS per sweep, time-to-eps and roofline fraction for every BASELINE.json config on one GPU
(the north star's reporting) -- library defaults, graph ingested once per config.

    python tools/all_configs.py [--configs 1,2,3,4,5] [--out gpurun_out/all_configs.json]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--out", default="gpurun_out/all_configs.json")
    args = ap.parse_args()
    import torch
    import paper_2206_09960_b200 as psi
    import psigen
    import bench
    peak, _ = bench._peaks()
    rows = []
    for k in [int(x) for x in args.configs.split(",")]:
        w = psigen.make_config(k)
        dev = [torch.from_numpy(a).cuda() for a in (w.row_ptr, w.followers, w.lam, w.mu)]
        with psi.PsiGraph(*dev) as g:
            inf = g.info()
            for _ in range(3):
                g.iterate(w.eps)
            times = []
            for _ in range(5):
                st, T, gap = g.iterate(w.eps)
                times.append(g.info()["iterate_ms"])
            g.time_sweep(3)
            hv, ti, fx = g.time_sweep(20)
            sweep = hv + ti + fx
            inf = g.info()
        byt = bench.algorithmic_bytes_per_sweep(w.n, w.m, inf["n_g"], inf["n_f"])
        r = {"config": k, "workload": psigen.CONFIG_NAMES[k], "N": w.n, "M": w.m, "eps": w.eps,
             "T": T, "time_to_eps_ms": round(statistics.median(times), 3),
             "solve_gteps": round(w.m * (T + 1) / statistics.median(times) / 1e6, 1),
             "sweep_ms": round(sweep, 4), "k_heavy_ms": round(hv, 4), "k_tiles_ms": round(ti, 4),
             "k_fix_ms": round(fx, 4), "sweep_gteps": round(w.m / sweep / 1e6, 1),
             "B_sweep": byt, "hbm_frac": round(byt / (sweep * 1e-3) / 1e9 / peak, 4),
             "n_heavy": inf["n_heavy"], "ingest_ms": round(inf["ingest_ms"], 1)}
        print(json.dumps(r), flush=True)
        rows.append(r)
        del dev
        torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    json.dump(rows, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
