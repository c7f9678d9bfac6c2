"""Config-2 step study (reading c9): final |x| and support recovery for fixed mu (fractions of the
config's mu) and the adaptive step (Algorithm 1).  Prints one line per setting."""
import sys
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
from paper_1802_04907_b200 import iht
from paper_1802_04907_b200.problem import build_pool
from workloads import gen as G

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
dev = torch.device('cuda:0')
p = G.config_problem(cfg)
pool, c_phi, prep, rows, row0 = build_pool(p, 0, 1, dev, False, shard="rows")
y_dev = torch.from_numpy(p.y[row0:row0 + rows]).to(dev)
true = set(p.x_idx.tolist())
for f, adaptive in [(1.0, False), (0.5, False), (0.25, False), (0.1, False), (1.0, True)]:
    mu = f * p.mu
    sol = iht.Solver(pool, p.s, p.n_iter, mu, p.b_y, p.seed, trace=True, adaptive=adaptive)
    sol.run(y_dev)
    torch.cuda.synchronize()
    idx, val, nnz = sol.trace_arrays()
    out = []
    for n in (9, 49, 99, 199):
        if n >= p.n_iter:
            continue
        k = int(nnz[n])
        if k < 0:
            out.append(f"it{n+1}: poisoned")
            continue
        sup = set(idx[n, :k].tolist())
        xe = np.zeros(p.N); xe[idx[n, :k].numpy()] = val[n, :k].numpy()
        xt = np.zeros(p.N); xt[p.x_idx] = p.x_val
        out.append(f"it{n+1}: hit {len(sup & true)}/{p.s} relerr {np.linalg.norm(xe - xt) / np.linalg.norm(xt):.3g}")
    print(f"config {cfg} mu={f} x {p.mu:.4g} adaptive={adaptive}: " + "; ".join(out), flush=True)
    sol.close()
