"""Which kernels and which host synchronisations happen inside one psi_iterate (+ get_psi),
seen by CUPTI through torch.profiler (no nsys in this image): evidence for the bench line's
gpu_launches and for "one host sync per solve" (SURVEY.md:333-336).

    python tools/launch_trace.py [--config 3] [--out gpurun_out/launch_trace.json]
"""
import argparse
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def trace(g, eps, out_dev):
    import torch
    from torch.profiler import profile, ProfilerActivity
    g.iterate(eps)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        st, T, gap = g.iterate(eps)
        g.get_psi(out=out_dev)
        torch.cuda.synchronize()
    kern = collections.Counter()
    api = collections.Counter()
    for e in prof.events():
        dt = str(getattr(e, "device_type", ""))
        if dt.endswith("CUDA"):
            kern[e.name] += 1
        elif e.name.startswith("cuda") or e.name.startswith("cu"):
            api[e.name] += 1
    return {"T": T, "kernels": dict(kern), "n_kernels": sum(kern.values()),
            "runtime_api": dict(api)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--out", default="gpurun_out/launch_trace.json")
    args = ap.parse_args()
    import torch
    import paper_2206_09960_b200 as psi
    import psigen
    w = psigen.make_config(args.config)
    dev = [torch.from_numpy(a).cuda() for a in (w.row_ptr, w.followers, w.lam, w.mu)]
    out = torch.empty(w.n, dtype=torch.float64, device="cuda")
    with psi.PsiGraph(*dev) as g:
        r = trace(g, w.eps, out)
        r["info"] = {k: g.info()[k] for k in ("n_heavy", "last_solver", "num_tiles")}
    print(json.dumps(r, indent=1))
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(r, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
