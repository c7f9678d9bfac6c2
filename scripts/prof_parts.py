"""Config-5-shaped forward_batched and threshold_batched timing (CUDA graph of 50 calls)
and config-4-shaped single-vector forward / threshold, for profiling."""
import sys
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
from paper_1802_04907_b200 import iht


def timeit(fn, reps=50):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


rng = np.random.default_rng(0)
which = sys.argv[1] if len(sys.argv) > 1 else "all"
if which in ("all", "c5"):
    M, N, B, s = 2304, 65536, 64, 64
    phi = torch.complex(torch.randn(M, N), torch.randn(M, N)).cuda()
    (F,) = iht.quantize(phi, 2, 0, 77, [3], float(iht.absmax(phi).item()))
    del phi
    xi = torch.from_numpy(np.stack([np.sort(rng.choice(N, s, replace=False)) for _ in range(B)]).astype(np.int32)).cuda()
    xv = torch.randn(B, s, device='cuda')
    nz = torch.full((B,), s, dtype=torch.int32, device='cuda')
    yh = torch.randn(B, iht.vec_len(M, 2), device='cuda')
    G = torch.randn(B, N, device='cuda')
    print(f"c5 forward_batched   {timeit(lambda: iht.forward_batched(F, xi, xv, nz, yh)):.1f} us")
    print(f"c5 threshold_batched {timeit(lambda: iht.threshold_batched(xi, xv, nz, G, 1e-3, s)):.1f} us")
if which in ("all", "c2"):
    N, s = 16384, 128
    xi = torch.from_numpy(np.sort(rng.choice(N, s, replace=False)).astype(np.int32)).cuda()
    xv = torch.randn(s, device='cuda')
    nz = torch.full((1,), s, dtype=torch.int32, device='cuda')
    g = torch.randn(N, device='cuda')
    print(f"c2 threshold         {timeit(lambda: iht.threshold(xi, xv, nz, g, 1.0, s)):.1f} us")
    (A2,) = [iht.new_copy(4096, N, 1, 2, 0, 77, 0, 1.0, device='cuda')]
    A2.codes.random_(0, 255)
    r2 = torch.randn(iht.vec_len(4096, 1), device='cuda')
    print(f"c2 adjoint           {timeit(lambda: iht.adjoint(A2, r2)):.1f} us")
if which in ("all", "c4"):
    M, N, s = 65536, 262144, 1024
    (F,) = [iht.new_copy(M, N, 1, 4, 0, 77, 0, 1.0, device='cuda')]
    F.codes.random_(0, 255)
    xi = torch.from_numpy(np.sort(rng.choice(N, s, replace=False)).astype(np.int32)).cuda()
    xv = torch.randn(s, device='cuda')
    nz = torch.full((1,), s, dtype=torch.int32, device='cuda')
    yh = torch.randn(iht.vec_len(M, 1), device='cuda')
    g = torch.randn(N, device='cuda')
    print(f"c4 forward           {timeit(lambda: iht.forward(F, xi, xv, nz, yh)):.1f} us")
    print(f"c4 threshold         {timeit(lambda: iht.threshold(xi, xv, nz, g, 1.0, s)):.1f} us")
