"""Config-4 forward (s = 1024 support columns of a 65536 x 262144 4-bit copy) and H_s
(N = 262144, s = 1024) timed alone with CUDA events (warm, back-to-back launches)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
from paper_1802_04907_b200 import iht
from paper_1802_04907_b200.problem import build_pool
from workloads import gen as G

dev = torch.device("cuda:0")
what = sys.argv[1] if len(sys.argv) > 1 else "forward"
rng = np.random.default_rng(4)


def timeit(fn, reps=50):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


N, s = 262144, 1024
xi = torch.from_numpy(np.sort(rng.choice(N, s, replace=False)).astype(np.int32)).to(dev)
xv = torch.from_numpy(rng.standard_normal(s).astype(np.float32)).to(dev)
nz = torch.tensor([s], dtype=torch.int32, device=dev)
if what == "forward":
    p = G.config_problem(4)
    p.K = 1
    pool, c, _, rows, row0 = build_pool(p, 0, 1, dev, False)
    yhat = torch.zeros(iht.vec_len(p.M, 1), device=dev)
    us = timeit(lambda: iht.forward(pool[0], xi, xv, nz, yhat))
    print(f"forward config 4 (IHT_FWD_WORDS={os.environ.get('IHT_FWD_WORDS', 'auto')}): {us:.1f} us", flush=True)
else:
    g = torch.from_numpy(rng.standard_normal(N).astype(np.float32)).to(dev)
    us = timeit(lambda: iht.threshold(xi, xv, nz, g, 0.5, s))
    print(f"threshold N={N} s={s} (IHT_THR_CL={os.environ.get('IHT_THR_CL', 'auto')}): {us:.1f} us", flush=True)
