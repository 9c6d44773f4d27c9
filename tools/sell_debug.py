import os, sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
import torch
import paper_2206_09960_b200 as psi
import oracle, psigen
from test_gpu_sell import random_graph
for seed in range(4):
    rng, rp, f, lam, mu = random_graph(seed)
    os.environ.update(PSI_SELL="1", PSI_SELL_SHIFT=str(5 + seed % 4), PSI_SELL_LMAX=str((2, 7, 40)[seed % 3]), PSI_SELL_PIECE=str((32, 33, 96)[seed % 3]))
    dev = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (rp, f, lam, mu)]
    try:
        with psi.PsiGraph(*dev) as g:
            info = g.info()
            print(seed, 'n', len(lam), 'info', {k: info[k] for k in ('n_f','sliced_ell','sell_long_rows','sell_pieces','sell_words','grid','block')}, flush=True)
            st, T, gap = g.iterate(0.0, 5)
            p = g.get_psi().cpu().numpy()
        ref = oracle.power_psi(rp, f, lam, mu, eps=0.0, max_iters=5)
        print(seed, 'T', T, 'err', oracle.max_rel_error(ref.psi, p), flush=True)
    except Exception as e:
        print(seed, 'ERROR', e, flush=True)
        break
