"""Config-4 adjoint (65536 x 262144, 4-bit, random codes) timed alone: back-to-back launches
alternating two copies (16 GiB > L2), CUDA events; GB/s of algorithmic bytes per launch.
Env knobs read by the library: IHT_ADJ_KR (rows per K-range), IHT_ADJ_RING (3 / 5 slots)."""
import os
import sys
import torch
sys.path.insert(0, "/root/repo")
from paper_1802_04907_b200 import iht

dev = torch.device("cuda:0")
bits = int(sys.argv[1]) if len(sys.argv) > 1 else 4
M, N = 65536, int(sys.argv[2]) if len(sys.argv) > 2 else 262144
A = [iht.new_copy(M, N, 1, bits, 0, 77, k, 1.0, device=dev) for k in range(2)]
for c in A:
    c.codes.random_(0, 255)
r = torch.randn(iht.vec_len(M, 1), device=dev)
g = torch.empty(N, device=dev)
for k in range(4):
    iht.adjoint(A[k % 2], r, out=g)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 40
e0.record()
for k in range(reps):
    iht.adjoint(A[k % 2], r, out=g)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / reps * 1e3
byts = M * N * bits / 8 + 4 * M + 4 * N
print(f"N {N} bits {bits} KR={os.environ.get('IHT_ADJ_KR', 'auto')} RING={os.environ.get('IHT_ADJ_RING', '3')}: "
      f"{us:.1f} us per adjoint, {byts / us / 1e3:.1f} GB/s")
