"""Config-4 H_s (N = 262144, s = 1024) on an iteration-shaped input (x = H_s of a previous a,
new g), timed alone: CUDA graph of 50 calls; checked once against numpy H_s.
IHT_THR_ONEPASS=0 times the three-launch path (T1 - T3)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
from paper_1802_04907_b200 import iht

dev = torch.device("cuda:0")
rng = np.random.default_rng(5)
N, s = 262144, 1024
a0 = rng.standard_normal(N).astype(np.float32)
order = np.lexsort((np.arange(N), -np.abs(a0)))[:s]
xi = np.sort(order).astype(np.int32)
xv = a0[xi]
g = (0.3 * rng.standard_normal(N)).astype(np.float32)
XI, XV = torch.from_numpy(xi).to(dev), torch.from_numpy(xv).to(dev)
NZ = torch.tensor([s], dtype=torch.int32, device=dev)
G = torch.from_numpy(g).to(dev)
oi, ov, on = iht.threshold(XI, XV, NZ, G, 1.0, s)
a = g.copy()
a[xi] += xv
ref = np.sort(np.lexsort((np.arange(N), -np.abs(a)))[:s])
assert int(on.item()) == s and oi[:s].cpu().numpy().tolist() == ref.tolist(), "H_s mismatch"
for _ in range(3):
    iht.threshold(XI, XV, NZ, G, 1.0, s)
torch.cuda.synchronize()
st = torch.cuda.Stream()
gr = torch.cuda.CUDAGraph()
with torch.cuda.stream(st):
    iht.threshold(XI, XV, NZ, G, 1.0, s)
    with torch.cuda.graph(gr, stream=st):
        for _ in range(50):
            iht.threshold(XI, XV, NZ, G, 1.0, s)
gr.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
gr.replay()
e1.record()
torch.cuda.synchronize()
print(f"H_s N={N} s={s} iteration-shaped (IHT_THR_ONEPASS={os.environ.get('IHT_THR_ONEPASS', '1')}): "
      f"{e0.elapsed_time(e1) / 50 * 1e3:.1f} us per call (graph of 50)")
