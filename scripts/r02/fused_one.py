"""One fused solve of config <cfg> (for ncu captures)."""
import sys

import torch

sys.path.insert(0, "/root/repo")
from paper_1802_04907_b200 import iht
from paper_1802_04907_b200.problem import build_pool
from workloads import gen as G

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n_iter = int(sys.argv[2]) if len(sys.argv) > 2 else 20
p = G.config_problem(cfg, K=2)
pool, c, _, rows, row0 = build_pool(p, 0, 1, torch.device("cuda:0"), False)
sol = iht.Solver(pool, p.s, n_iter, p.mu, p.b_y, p.seed)
assert sol.fused
sol.run(torch.from_numpy(p.y).cuda())
torch.cuda.synchronize()
print("done", cfg, n_iter)
