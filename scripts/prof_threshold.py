"""Threshold phase timeline (IHT_THR_TL=1): config-5-like (64 x 65536, s = 64) and
config-2-like (1 x 16384, s = 128) inputs, a = x + mu g with Gaussian g and an s-sparse x
of magnitude ~3 sigma.  Prints the per-phase globaltimer offsets (ns) from stderr."""
import sys

import numpy as np
import torch

sys.path.insert(0, '/root/repo')
from paper_1802_04907_b200 import iht

for (B, N, s) in [(64, 65536, 64), (1, 16384, 128), (1, 65536, 64)]:
    rng = np.random.default_rng(N)
    g = torch.from_numpy(rng.standard_normal((B, N)).astype(np.float32)).cuda()
    xi = np.stack([np.sort(rng.choice(N, s, replace=False)) for _ in range(B)]).astype(np.int32)
    xv = (3.0 * np.sign(rng.standard_normal((B, s)))).astype(np.float32)
    nz = np.full(B, s, np.int32)
    print(f"B={B} N={N} s={s}", file=sys.stderr, flush=True)
    for _ in range(3):
        iht.threshold_batched(torch.from_numpy(xi).cuda(), torch.from_numpy(xv).cuda(), torch.from_numpy(nz).cuda(),
                              g, 0.25, s)
    torch.cuda.synchronize()
