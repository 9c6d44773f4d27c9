"""e2e variance diagnosis: repeated build/iterate/get/destroy at a config with the stream-ordered
pool's reserved / used bytes printed around every step (cuda-python runtime API).

    python tools/e2e_pool_diag.py [--config 5] [--reps 8]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pool_bytes():
    from cuda.bindings import runtime as rt
    _, pool = rt.cudaDeviceGetDefaultMemPool(0)
    _, res = rt.cudaMemPoolGetAttribute(pool, rt.cudaMemPoolAttr.cudaMemPoolAttrReservedMemCurrent)
    _, used = rt.cudaMemPoolGetAttribute(pool, rt.cudaMemPoolAttr.cudaMemPoolAttrUsedMemCurrent)
    return int(res) / 2**30, int(used) / 2**30


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
        r0 = pool_bytes()
        t0 = time.perf_counter()
        g = psi.PsiGraph(*host)
        t1 = time.perf_counter()
        r1 = pool_bytes()
        g.iterate(w.eps)
        g.get_psi(out=out)
        t2 = time.perf_counter()
        g.close()
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        print(f"rep {r}: build {1e3*(t1-t0):7.1f}  iterate+get {1e3*(t2-t1):6.1f}  destroy {1e3*(t3-t2):6.1f} ms"
              f"  pool reserved/used GiB before {r0[0]:.1f}/{r0[1]:.1f} after build {r1[0]:.1f}/{r1[1]:.1f}",
              flush=True)


if __name__ == "__main__":
    main()
