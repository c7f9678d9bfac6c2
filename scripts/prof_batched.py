"""Config-5-size batched adjoint (tcgen05) for profiling: 2304x65536 complex, 2-bit, B=64."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
from paper_1802_04907_b200 import iht
rng = np.random.default_rng(0)
M, N, B = 2304, 65536, 64
phi = torch.complex(torch.randn(M, N), torch.randn(M, N)).cuda()
c = float(iht.absmax(phi).item())
(A,) = iht.quantize(phi, 2, 0, 77, [3], c)
del phi
R = torch.randn(B, iht.vec_len(M, 2), device='cuda')
for _ in range(5):
    G = iht.adjoint_batched(A, R)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50):
    G = iht.adjoint_batched(A, R)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 50
flops = 2 * 65536 * 4608 * 64
print(f"batched adjoint {ms*1e3:.1f} us/call, useful {flops/ms/1e9:.1f} TFLOP/s (2 N R B), codes {65536*4608/4/ms/1e6:.1f} GB/s")
