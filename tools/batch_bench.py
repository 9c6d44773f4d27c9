"""Multi-profile batch at a BASELINE config: per-sweep device time of the
four-profile sweep, time-to-eps of k profiles, against the single-profile sweep on the same
graph.   python tools/batch_bench.py [--config 5] [--k 4] [--out gpurun_out/batch.json]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--k", type=int, default=4)
    ap.add_argument("--out", default="gpurun_out/batch.json")
    a = ap.parse_args()
    import numpy as np
    import torch
    import paper_2206_09960_b200 as psi
    import psigen
    w = psigen.make_config(a.config)
    n = w.row_ptr.size - 1
    m = w.followers.size
    lam, mu = psigen.activity_profiles(n, a.k, "lognormal", pure_posters=(a.config == 5))
    lam[0], mu[0] = w.lam, w.mu
    dev = [torch.from_numpy(x).cuda() for x in (w.row_ptr, w.followers)]
    L, M = torch.from_numpy(lam).cuda(), torch.from_numpy(mu).cuda()
    out = {"config": a.config, "N": n, "M": m, "k": a.k}
    with psi.PsiGraph(dev[0], dev[1], L, M) as g:
        out["ingest_ms"] = round(g.info()["ingest_ms"], 1)
        g.time_sweep_batch(3)
        out["batch_sweep_ms"] = round(g.time_sweep_batch(20), 4)
        ts = []
        for _ in range(4):
            st, T, gap = g.iterate(w.eps)
            ts.append(g.info()["iterate_ms"])
        Tp, gp = g.profile_stats()
        out["time_to_eps_ms"] = round(sorted(ts)[len(ts) // 2], 3)
        out["T_profiles"] = Tp.tolist()
    torch.cuda.empty_cache()
    with psi.PsiGraph(dev[0], dev[1], L[0].contiguous(), M[0].contiguous()) as g:
        g.time_sweep(3)
        h, t, f = g.time_sweep(20)
        out["single_sweep_ms"] = round(h + t + f, 4)
        ts = []
        for _ in range(4):
            g.iterate(w.eps)
            ts.append(g.info()["iterate_ms"])
        out["single_time_to_eps_ms"] = round(sorted(ts)[len(ts) // 2], 3)
    groups = (a.k + 3) // 4
    out["profile_gteps_batch"] = round(4 * m / (out["batch_sweep_ms"] * 1e6), 1)
    out["gteps_single"] = round(m / (out["single_sweep_ms"] * 1e6), 1)
    out["speedup_per_profile_sweep"] = round(4 * out["single_sweep_ms"] / out["batch_sweep_ms"], 2)
    out["groups"] = groups
    print(json.dumps(out))
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
