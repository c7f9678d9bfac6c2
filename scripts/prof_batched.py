"""Config-5-size batched adjoint (tcgen05) timing: 2304x65536 complex, 2-bit, B=64.
Buffers preallocated, 50 calls captured in one CUDA graph (no host overhead in the timing).
Prints per-call time; the ncu launch list splits it into the limb-prep and GEMM kernels."""
import ctypes
import sys

import torch

sys.path.insert(0, '/root/repo')
from paper_1802_04907_b200 import iht
from paper_1802_04907_b200._lib import check, load

M, N, B = 2304, 65536, int(sys.argv[1]) if len(sys.argv) > 1 else 64
bits = int(sys.argv[2]) if len(sys.argv) > 2 else 2
torch.manual_seed(0)
phi = torch.complex(torch.randn(M, N), torch.randn(M, N)).cuda()
c = float(iht.absmax(phi).item())
(A,) = iht.quantize(phi, bits, 0, 77, [3], c)
del phi
R = torch.randn(B, iht.vec_len(M, 2), device='cuda')
lib = load()
wsb = lib.iht_adjoint_batched_ws_bytes(ctypes.byref(A.desc), B)
ws = torch.empty(wsb, dtype=torch.uint8, device='cuda')
G = torch.empty((B, N), device='cuda')


def call():
    check(lib.iht_adjoint_batched(ctypes.byref(A.desc), ctypes.c_void_p(R.data_ptr()), B,
                                  ctypes.c_void_p(G.data_ptr()), ctypes.c_void_p(ws.data_ptr()), wsb,
                                  ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)), "adj")


for _ in range(3):
    call()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):
        for _ in range(50):
            call()
torch.cuda.synchronize()
g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(4):
    g.replay()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 200
flops = 2 * N * 4608 * B
print(f"B={B} bits={bits}: batched adjoint {ms*1e3:.1f} us/call (graph), useful {flops/ms/1e9:.1f} TOP/s (2 N R B), "
      f"codes {N*4608*bits/8/ms/1e6:.1f} GB/s")
