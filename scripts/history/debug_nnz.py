"""Debug: does the solver's final nnz go negative (poisoned) on config 2/3? profile on/off,
device run vs host run; prints the first traced iteration with nnz < 0."""
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
for profile in (False,):
    for trace in (True,):
        sol = iht.Solver(pool, p.s, p.n_iter, p.mu, p.b_y, p.seed, profile=profile, trace=trace)
        res = []
        for _ in range(4):
            sol.run(y_dev)
            torch.cuda.synchronize()
            res.append(int(sol.out_nnz.cpu()[0]))
        line = f"profile={profile} trace={trace}: device nnz {res}"
        if trace:
            idx, val, nnz = sol.trace_arrays()
            bad = np.nonzero(nnz.numpy() < 0)[0]
            line += f" first bad iter {bad[:3].tolist()} nnz head {nnz[:5].tolist()}"
            mx = np.abs(val.numpy()).max(axis=1)
            line += f" max|x| at 0,50,100,150,190,194: {[float(mx[i]) for i in (0, 50, 100, 150, 190, 194)]}"
        y_pin = torch.from_numpy(p.y[row0:row0 + rows].copy()).pin_memory()
        oi = torch.empty((p.s,), dtype=torch.int32).pin_memory()
        ov = torch.empty((p.s,), dtype=torch.float32).pin_memory()
        on = torch.empty(1, dtype=torch.int32).pin_memory()
        try:
            sol.run_host(y_pin, oi, ov, on)
            line += f" host nnz {int(on[0])}"
        except Exception as e:
            line += f" host FAIL {e}"
        print(line, flush=True)
        sol.close()
