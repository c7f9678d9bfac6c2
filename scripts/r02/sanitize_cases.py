"""Small launches of every hand-written kernel for compute-sanitizer (memcheck / racecheck /
synccheck): quantiser, forward, int8-MMA adjoint (one and two K-ranges), fused cluster
threshold, tcgen05 batched adjoint, batched forward/threshold, the fused persistent solver,
the per-step solver graph.  Results are checked loosely (finite, right sizes); parity is the
test suite's job."""
import sys

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
from paper_1802_04907_b200 import iht

dev = torch.device("cuda:0")
rng = np.random.default_rng(0)
which = sys.argv[1] if len(sys.argv) > 1 else "all"


def t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


M, N, s = 512, 1040, 24
phi = rng.standard_normal((M, N)).astype(np.float32)
c = float(np.abs(phi).max())
pool = iht.quantize(t(phi), 2, 0, 7, [0, 1], c)
x_idx = np.sort(rng.choice(N, s, replace=False)).astype(np.int32)
x_val = rng.standard_normal(s).astype(np.float32)
nz = t(np.array([s], np.int32))
yhat = t(np.concatenate([rng.standard_normal(M), np.zeros(iht.vec_len(M, 1) - M)]).astype(np.float32))
if which in ("all", "forward"):
    r = iht.forward(pool[1], t(x_idx), t(x_val), nz, yhat)
if which in ("all", "adjoint"):
    g = iht.adjoint(pool[0], yhat)
    big = iht.quantize(t(rng.standard_normal((33000, 48)).astype(np.float32)), 4, 0, 7, [0], 5.0)   # 2 K-ranges
    g2 = iht.adjoint(big[0], t(rng.standard_normal(iht.vec_len(33000, 1)).astype(np.float32)))
if which in ("all", "threshold"):
    oi, ov, on = iht.threshold(t(x_idx), t(x_val), nz, t(rng.standard_normal(N).astype(np.float32)), 0.5, s)
if which in ("all", "batched"):
    B = 8
    R = t(rng.standard_normal((B, iht.vec_len(M, 1))).astype(np.float32))
    G = iht.adjoint_batched(pool[0], R)
    xi = t(np.stack([x_idx] * B))
    xv = t(np.stack([x_val] * B))
    nzb = t(np.full(B, s, np.int32))
    Rf = iht.forward_batched(pool[1], xi, xv, nzb, R)
    oi, ov, on = iht.threshold_batched(xi, xv, nzb, G, 0.5, s)
if which in ("all", "fused", "solver"):
    y = t((phi.astype(np.float64) @ np.where(np.isin(np.arange(N), x_idx), 1.0, 0.0)).astype(np.float32))
    for fused in (["force"] if which == "fused" else [False] if which == "solver" else ["force", False]):
        sol = iht.Solver(pool, s, 4, 0.3, 8, 7, fused=fused)
        sol.run(y)
        torch.cuda.synchronize()
        sol.close()
torch.cuda.synchronize()
print("sanitize cases done:", which, "library:", iht._lib.load()._name)
