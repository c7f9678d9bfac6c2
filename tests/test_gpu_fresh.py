"""GPU parity of NEXT-2 (fresh copies drawn on the fly from the fp32 Phi, no stored codes)
against the oracle, whose CopyPool with K = 2 n* is exactly Algorithm 1's 2 n* independent
copies.

* codes: the adjoint of a unit vector e_m returns sigma (2 code_{m,:} - (L-1)), exact in
  fp32, so comparing it with the oracle's codes of copy k checks every code of row m
  bit for bit;
* adjoint / forward within 1e-4 of the oracle for the same copy id;
* the fresh solver follows the oracle's K = 2 n* trajectory (near-tie rule as elsewhere).
"""
import numpy as np
import pytest
import torch

from oracle import iht as OI
from oracle import quantize as OQ
from paper_1802_04907_b200 import iht
from workloads import gen as G

from helpers import rel_l2, stack, unstack

pytestmark = pytest.mark.gpu
TOL = 1e-4
SEED = 0x1802_0490_7F5


def _dev():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch.device("cuda:0")


def _to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(_dev())


def _phi(M, N, cplx, seed):
    rng = np.random.default_rng(seed)
    if cplx:
        return (rng.standard_normal((M, N)) + 1j * rng.standard_normal((M, N))).astype(np.complex64)
    return rng.standard_normal((M, N)).astype(np.float32)


@pytest.mark.parametrize("M,N,cplx,bits,mode", [(300, 1001, False, 2, 0), (256, 1024, False, 4, 0),
                                                 (100, 777, True, 2, 0), (513, 37, False, 8, 1)])
def test_fresh_codes_exact_via_unit_vectors(M, N, cplx, bits, mode):
    phi = _phi(M, N, cplx, seed=M)
    c = OQ.scale_c(phi)
    F = iht.fresh_phi(_to_dev(phi), bits, mode, SEED, float(c))
    L = OQ.num_levels(bits, mode)
    sigma = np.float32(np.float32(c) / np.float32(L - 1))
    planes = 2 if cplx else 1
    for k in (0, 5, 399):
        codes, _ = OQ.quantize_matrix(phi, bits, mode, SEED, k, c=c)
        for m in (0, M // 2, M - 1):
            for p in range(planes):
                e = np.zeros(planes * ((M + 255) // 256 * 256), np.float32)
                e[p * ((M + 255) // 256 * 256) + m] = 1.0
                g = iht.adjoint_fresh(F, k, _to_dev(e)).cpu().numpy()
                q = (2 * codes[p, m].astype(np.int64) - (L - 1)).astype(np.float32)
                np.testing.assert_array_equal(g, (sigma * q).astype(np.float32))


@pytest.mark.parametrize("M,N,cplx,bits", [(300, 1001, False, 2), (2304, 3000, True, 2), (4500, 777, False, 4)])
def test_fresh_adjoint_forward_parity(M, N, cplx, bits):
    phi = _phi(M, N, cplx, seed=N)
    c = OQ.scale_c(phi)
    F = iht.fresh_phi(_to_dev(phi), bits, 0, SEED, float(c))
    planes = 2 if cplx else 1
    rng = np.random.default_rng(3)
    for k in (2, 17):
        Ad = OQ.dequantize(OQ.quantize_matrix(phi, bits, 0, SEED, k, c=c)[0], c, bits, 0)
        r = rng.standard_normal(M) + (1j * rng.standard_normal(M) if cplx else 0)
        r32 = stack(r, M).astype(np.float32)
        g = iht.adjoint_fresh(F, k, _to_dev(r32)).cpu().numpy()
        assert rel_l2(g, OI.adjoint(Ad, unstack(r32, M, planes))) < TOL
        s = 23
        xi = np.sort(rng.choice(N, s, replace=False)).astype(np.int32)
        xv = rng.standard_normal(s).astype(np.float32)
        yh = stack(rng.standard_normal(M) + (1j * rng.standard_normal(M) if cplx else 0), M).astype(np.float32)
        rr = iht.forward_fresh(F, k, _to_dev(xi), _to_dev(xv), _to_dev(np.array([s], np.int32)), _to_dev(yh))
        ref = OI.forward(Ad, xi, xv.astype(np.float64), unstack(yh, M, planes))
        assert rel_l2(unstack(rr.cpu().numpy(), M, planes), ref) < TOL


CASES = {
    "config1": lambda: G.config_problem(1, K=40),
    "radio": lambda: G.radio_problem(cfg_id=71, A=12, grid=48, n_src=10, n_iter=20, K=40),
}


@pytest.mark.parametrize("case", list(CASES))
def test_fresh_solver_matches_oracle_2n_copies(case):
    p = CASES[case]()
    n_iter = 20
    ref = OI.qniht(p.phi, p.y, p.s, n_iter, p.mu, p.b_phi, p.b_y, p.seed, 2 * n_iter)
    F = iht.fresh_phi(_to_dev(p.phi), p.b_phi, 0, p.seed, float(OQ.scale_c(p.phi)))
    sol = iht.Solver(F, p.s, n_iter, p.mu, p.b_y, p.seed, trace=True)
    sol.run(_to_dev(p.y))
    torch.cuda.synchronize()
    idx, val, nnz = sol.trace_arrays()
    checked = 0
    for n, rec in enumerate(ref.trace):
        a = np.sort(np.abs(rec.a))[::-1]
        if rec.margin <= 1e-5 * max(a[p.s - 1], 1e-30):
            break
        k = int(nnz[n])
        assert idx[n, :k].tolist() == rec.x_idx.tolist(), f"iteration {rec.n}"
        assert rel_l2(val[n, :k].numpy(), rec.x_val, floor=1e-30) < TOL
        checked += 1
    assert checked >= min(n_iter, 10), checked
    sol.close()
