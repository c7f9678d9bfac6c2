"""Fused kernel phase timeline (IHT_FUSED_TL=<cta>): configs 1-3, CTA 0 and CTA 147."""
import os
import sys

import torch

sys.path.insert(0, "/root/repo")
from paper_1802_04907_b200 import iht
from paper_1802_04907_b200.problem import build_pool
from workloads import gen as G

dev = torch.device("cuda:0")
for cfg in [int(c) for c in (sys.argv[1:] or ["1", "2", "3"])]:  # TL_CTAS=-1: every CTA
    p = G.config_problem(cfg)
    pool, c, _, rows, row0 = build_pool(p, 0, 1, dev, False)
    y = torch.from_numpy(p.y).to(dev)
    for cta in os.environ.get("TL_CTAS", "0,147").split(","):
        os.environ["IHT_FUSED_TL"] = cta
        sol = iht.Solver(pool, p.s, p.n_iter, p.mu, p.b_y, p.seed)
        for _ in range(2):
            sol.run(y)
        torch.cuda.synchronize()
        print(f"config {cfg} cta {cta}:", file=sys.stderr, flush=True)
        sol.close()
    os.environ.pop("IHT_FUSED_TL")
    del pool
    torch.cuda.empty_cache()
