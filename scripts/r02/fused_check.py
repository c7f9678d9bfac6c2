"""Quick GPU check of the fused persistent solver against the per-step kernels and the oracle
(small cases), plus per-iteration timings of both paths on configs 1-3."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
sys.path.insert(0, "/root/repo/tests")
from oracle import iht as OI
from oracle import quantize as OQ
from paper_1802_04907_b200 import iht
from paper_1802_04907_b200.problem import build_pool
from workloads import gen as G
from helpers import check_trajectory

dev = torch.device("cuda:0")


def pool_of(p, K):
    c = OQ.scale_c(p.phi)
    return iht.quantize(torch.from_numpy(p.phi).to(dev), p.b_phi, 0, p.seed, list(range(K)), float(c))


cases = {
    "config1": G.config_problem(1, K=40),
    "gauss2bit": G.gaussian_problem(1024, 4096, 40, cfg_id=21, values="sign", b_phi=2, n_iter=30, mu=0.15, K=60),
    "radio": G.radio_problem(cfg_id=23, A=12, grid=48, n_src=10, n_iter=30, K=60),
    "gauss8bit": G.gaussian_problem(700, 3001, 20, cfg_id=22, b_phi=8, n_iter=25, K=4),
}
for name, p in cases.items():
    n_iter = min(p.n_iter, 20)
    K = min(p.K, 2 * n_iter)
    pool = pool_of(p, K)
    ref = OI.qniht(p.phi, p.y, p.s, n_iter, p.mu, p.b_phi, p.b_y, p.seed, K)
    y = torch.from_numpy(p.y).to(dev)
    for fused in (True, False):
        sol = iht.Solver(pool, p.s, n_iter, p.mu, p.b_y, p.seed, trace=True, fused="force" if fused else False)
        sol.run(y)
        torch.cuda.synchronize()
        idx, val, nnz = sol.trace_arrays()
        try:
            chk = check_trajectory(ref.trace, idx, val, nnz, p.s, 1e-4)
            msg = f"{chk}/{n_iter} ok"
        except AssertionError as e:
            msg = f"FAIL {e}"
        print(f"{name} fused={fused} is_fused={sol.fused}: {msg}", flush=True)
        sol.close()

for cfg in (1, 2, 3):
    p = G.config_problem(cfg)
    pool, c, _, rows, row0 = build_pool(p, 0, 1, dev, False)
    y = torch.from_numpy(p.y).to(dev)
    for fused in (True, False):
        sol = iht.Solver(pool, p.s, p.n_iter, p.mu, p.b_y, p.seed, fused="force" if fused else False)
        for _ in range(3):
            sol.run(y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            sol.run(y)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(f"config {cfg} fused={sol.fused}: {ms * 1e3 / p.n_iter:.2f} us/iter, {p.n_iter * 1e3 / ms:.0f} iter/s",
              flush=True)
        sol.close()
    del pool
    torch.cuda.empty_cache()
