import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from oracle import quantize as OQ, iht as OI
from paper_1802_04907_b200 import iht
from helpers import stack, rel_l2
from workloads import gen as G
def run(M, N, B, bits, cplx, seed=0):
    rng = np.random.default_rng(seed)
    phi = (rng.standard_normal((M, N)) + (1j * rng.standard_normal((M, N)) if cplx else 0)).astype(np.complex64 if cplx else np.float32)
    c = OQ.scale_c(phi)
    (A,) = iht.quantize(torch.from_numpy(phi).cuda(), bits, 0, 77, [3], float(c))
    Ad = OQ.dequantize(OQ.quantize_matrix(phi, bits, 0, 77, 3, c=c)[0], c, bits, 0)
    R = np.stack([stack(rng.standard_normal(M) + (1j * rng.standard_normal(M) if cplx else 0), M) for _ in range(B)]).astype(np.float32)
    G = iht.adjoint_batched(A, torch.from_numpy(R).cuda())
    torch.cuda.synchronize()
    Gh = G.cpu().numpy()
    planes = 2 if cplx else 1
    errs = []
    for b in range(B):
        rb = R[b]
        rp = (M + 255)//256*256
        r = rb[:M] + (1j * rb[rp:rp+M] if cplx else 0)
        ref = OI.adjoint(Ad, r.astype(np.complex128 if cplx else np.float64))
        errs.append(rel_l2(Gh[b], ref))
    print(M, N, B, bits, cplx, "max rel err", max(errs), "first", errs[:3], flush=True)
    # timing
    Rt = torch.from_numpy(R).cuda()
    for _ in range(3): iht.adjoint_batched(A, Rt)
    torch.cuda.synchronize(); t=time.time()
    for _ in range(20): iht.adjoint_batched(A, Rt)
    torch.cuda.synchronize(); dt=(time.time()-t)/20
    print("  time/call %.1f us" % (dt*1e6), flush=True)
run(300, 500, 8, 2, False)
run(144, 2304, 8, 2, True)
run(1000, 1000, 16, 4, False)
run(1000, 700, 16, 8, False)
run(2304, 65536, 64, 2, True)
