"""GPU parity of NEXT-3 (the radio Phi computed on the fly, paper "Computing Phi on the
fly") against the oracle's dense products over the stored Phi of
workloads.gen.radio_problem (reading c16).

* full precision: Re(Phi^H r) within 1e-5 relative l2 of the float64 dense product;
* quantised in registers (copy k): within 1e-4 of the oracle adjoint over the stored-copy
  codes of the same copy (the on-the-fly fp32 entries match the stored complex64 Phi to
  about an ulp, so at most a handful of codes can differ);
* zero r gives zero g.
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


def _dev():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch.device("cuda:0")


def _uv(p):
    pos, lam = p.meta["antennas"], p.meta["wavelength"]
    A = pos.shape[0]
    b = (pos[:, None, :] - pos[None, :, :]).reshape(A * A, 2)
    return (torch.from_numpy(np.ascontiguousarray(b[:, 0] / lam)).to(_dev()),
            torch.from_numpy(np.ascontiguousarray(b[:, 1] / lam)).to(_dev()))


@pytest.mark.parametrize("A,grid", [(12, 48), (20, 64), (48, 256)])
def test_radio_on_the_fly_full_precision(A, grid):
    p = G.radio_problem(cfg_id=81, A=A, grid=grid, n_src=5, n_iter=1, K=2)
    u, v = _uv(p)
    rng = np.random.default_rng(A)
    r = rng.standard_normal(p.M) + 1j * rng.standard_normal(p.M)
    r32 = stack(r, p.M).astype(np.float32)
    g = iht.adjoint_radio(u, v, grid, torch.from_numpy(r32).to(_dev())).cpu().numpy()
    ref = OI.adjoint(p.phi.astype(np.complex128), unstack(r32, p.M, 2))
    assert rel_l2(g, ref) < 1e-5, rel_l2(g, ref)
    z = iht.adjoint_radio(u, v, grid, torch.zeros(len(r32), device=_dev()))
    assert torch.count_nonzero(z) == 0


@pytest.mark.parametrize("A,grid,bits", [(12, 48, 2), (20, 64, 4), (48, 128, 2)])
def test_radio_on_the_fly_quantised(A, grid, bits):
    p = G.radio_problem(cfg_id=82, A=A, grid=grid, n_src=5, n_iter=1, K=2)
    u, v = _uv(p)
    c = OQ.scale_c(p.phi)
    seed, k = 0x5EED_0003, 7
    rng = np.random.default_rng(grid)
    r = rng.standard_normal(p.M) + 1j * rng.standard_normal(p.M)
    r32 = stack(r, p.M).astype(np.float32)
    g = iht.adjoint_radio(u, v, grid, torch.from_numpy(r32).to(_dev()), bits=bits, seed=seed, copy_id=k,
                          scale_c=float(c)).cpu().numpy()
    Ad = OQ.dequantize(OQ.quantize_matrix(p.phi, bits, 0, seed, k, c=c)[0], c, bits, 0)
    ref = OI.adjoint(Ad, unstack(r32, p.M, 2))
    assert rel_l2(g, ref) < 1e-4, rel_l2(g, ref)
