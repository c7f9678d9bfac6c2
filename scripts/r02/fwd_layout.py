"""Config-4 forward timing (s = 1024 support columns of a 65536 x 262144 4-bit copy, random
codes), L2 flushed before every call, for each words-per-CTA variant (IHT_FWD_WORDS).
r02 g43 also timed a column-contiguous address pattern (IHT_FWD_STRIPS, since removed): the
same 30.7 us as the tiled layout.  Timing only: codes are random."""
import sys
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
from paper_1802_04907_b200 import iht

dev = torch.device("cuda:0")
rng = np.random.default_rng(4)
M, N, s = 65536, 262144, 1024
F = iht.new_copy(M, N, 1, 4, 0, 77, 0, 1.0, device=dev)
F.codes.random_(0, 255)
xi = torch.from_numpy(np.sort(rng.choice(N, s, replace=False)).astype(np.int32)).to(dev)
xv = torch.from_numpy(rng.standard_normal(s).astype(np.float32)).to(dev)
nz = torch.tensor([s], dtype=torch.int32, device=dev)
yhat = torch.zeros(iht.vec_len(M, 1), device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
ts = []
for rep in range(30):
    flush.fill_(rep)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    iht.forward(F, xi, xv, nz, yhat)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
print(sys.argv[1:], "median us (L2 flushed)", round(float(np.median(ts[3:])), 2), "min", round(min(ts[3:]), 2))
