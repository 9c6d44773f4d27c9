"""Overlapped-plan timing at C5: the pair concurrently vs its kernels one after the other."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2206_09960_b200 as psi, psigen
w = psigen.make_config(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
dev = [torch.from_numpy(a).cuda() for a in (w.row_ptr, w.followers, w.lam, w.mu)]
for ovl in ("0", "1"):
    os.environ["PSI_OVERLAP"] = ovl
    with psi.PsiGraph(*dev) as g:
        for ser in ("0", "1"):
            os.environ["PSI_OVL_SERIAL"] = ser
            g.time_sweep(3)
            print(f"OVERLAP={ovl} SERIAL={ser}: heavy %.3f tiles %.3f fix %.3f" % g.time_sweep(10),
                  g.info()["overlapped"], flush=True)
