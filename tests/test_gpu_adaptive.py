"""GPU parity of Algorithm 1's adaptive step (cfg.step_mode = 1)
against oracle.iht.qniht_adaptive, through the solver's C ABI.

Per iteration: the accepted step mu within 1e-4 relative (1e-3 on the tensor-core batched
path), the shrink count and the support identical, x within the path's tolerance -- up
to the first iteration whose decisions sit on a knife edge in the oracle (selection
margin below 1e-5 (1e-3 batched) of |a|_(s), or an acceptance test within 1e-4 (1e-3) of
mu), after which the fp32 and fp64 trajectories may legitimately part.  The captured
graph (conditional WHILE node) and the host-driven loop give bit-identical results.
"""
import numpy as np
import pytest
import torch

from oracle import iht as OI
from oracle import quantize as OQ
from paper_1802_04907_b200 import iht
from workloads import gen as G

from helpers import rel_l2

pytestmark = pytest.mark.gpu


def _dev():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch.device("cuda:0")


def _to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(_dev())


def _pool(phi, bits, K, seed):
    return iht.quantize(_to_dev(phi), bits, 0, seed, list(range(K)), float(OQ.scale_c(phi)))


def _clean(rec, tol_sel, tol_acc):
    return rec.select_margin > tol_sel and rec.accept_margin > tol_acc


def _compare(recs, idx, val, nnz, mu, sh, tol_x, tol_mu, tol_sel, tol_acc):
    checked = 0
    for n, rec in enumerate(recs):
        if not _clean(rec, tol_sel, tol_acc):
            return checked, False
        k = int(nnz[n])
        assert idx[n, :k].tolist() == rec.x_idx.tolist(), f"iteration {rec.n}: support"
        assert int(sh[n]) == rec.shrinks, f"iteration {rec.n}: shrinks {int(sh[n])} vs {rec.shrinks}"
        assert abs(float(mu[n]) - rec.mu) <= tol_mu * rec.mu, f"iteration {rec.n}: mu {float(mu[n])} vs {rec.mu}"
        assert rel_l2(val[n, :k], rec.x_val, floor=1e-30) < tol_x, f"iteration {rec.n}: x"
        checked += 1
    return checked, True


CASES = {
    "gauss4bit": lambda: G.gaussian_problem(256, 1024, 16, cfg_id=61, b_phi=4, n_iter=15, K=30),
    "gauss2bit": lambda: G.gaussian_problem(1024, 4096, 40, cfg_id=63, values="sign", b_phi=2, n_iter=12, K=24),
    "radio": lambda: G.radio_problem(cfg_id=63, A=12, grid=48, n_src=10, n_iter=12, K=24),
}


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("graph", [True, False])
def test_adaptive_solver_matches_oracle(case, graph):
    p = CASES[case]()
    xi, xv, recs = OI.qniht_adaptive(p.phi, p.y, p.s, p.n_iter, p.b_phi, p.b_y, p.seed, p.K, mu_fallback=p.mu)
    pool = _pool(p.phi, p.b_phi, p.K, p.seed)
    sol = iht.Solver(pool, p.s, p.n_iter, p.mu, p.b_y, p.seed, trace=True, use_graph=graph, adaptive=True)
    sol.run(_to_dev(p.y))
    torch.cuda.synchronize()
    idx, val, nnz = sol.trace_arrays()
    mu, sh = sol.steps()
    checked, clean = _compare(recs, idx.numpy(), val.numpy(), nnz.numpy(), mu.numpy(), sh.numpy(), 1e-4, 1e-4, 1e-5,
                              1e-4)
    assert checked >= min(10, p.n_iter), checked
    if clean:
        assert idx[-1, :int(nnz[-1])].tolist() == xi.tolist()
    sol.close()


def test_adaptive_graph_equals_host_loop_and_shrinks():
    """A scaled Gaussian operator makes first proposals overshoot: the shrink loop runs on
    the GPU (conditional WHILE node) exactly as in the host-driven loop."""
    rng = np.random.default_rng(5)
    M, N, s = 128, 512, 12
    phi = (3.0 * rng.standard_normal((M, N)) / np.sqrt(M)).astype(np.float32)
    x = np.zeros(N)
    x[np.sort(rng.choice(N, s, replace=False))] = rng.standard_normal(s)
    y = (phi.astype(np.float64) @ x).astype(np.float32)
    K, n_iter, seed = 20, 10, 0x5EED
    pool = _pool(phi, 8, K, seed)
    outs = []
    for graph in (True, False):
        sol = iht.Solver(pool, s, n_iter, 1.0, 8, seed, trace=True, use_graph=graph, adaptive=True)
        sol.run(_to_dev(y))
        torch.cuda.synchronize()
        outs.append((sol.trace_arrays(), sol.steps()))
        sol.close()
    (i0, v0, n0), (m0, s0) = outs[0]
    (i1, v1, n1), (m1, s1) = outs[1]
    assert torch.equal(i0, i1) and torch.equal(v0, v1) and torch.equal(n0, n1)
    assert torch.equal(m0, m1) and torch.equal(s0, s1)
    assert int(s0.sum()) > 0, "no proposal was rejected: the shrink loop was not exercised"
    xi, xv, recs = OI.qniht_adaptive(phi, y, s, n_iter, 8, 8, seed, K, mu_fallback=1.0)
    checked, _ = _compare(recs, i0.numpy(), v0.numpy(), n0.numpy(), m0.numpy(), s0.numpy(), 1e-4, 1e-4, 1e-5, 1e-4)
    assert checked >= 1


def test_adaptive_batched_matches_oracle():
    B = 8
    p = G.radio_problem(cfg_id=64, A=12, grid=48, n_src=8, n_iter=10, K=20, batch=B)
    Y = np.ascontiguousarray(p.meta["batch_y"].T)
    pool = _pool(p.phi, p.b_phi, p.K, p.seed)
    sol = iht.Solver(pool, p.s, p.n_iter, p.mu, p.b_y, p.seed, trace=True, nrhs=B, adaptive=True)
    sol.run(_to_dev(Y))
    torch.cuda.synchronize()
    idx, val, nnz = sol.trace_arrays()
    mu, sh = sol.steps()
    opool = OI.CopyPool(p.phi, p.b_phi, 0, p.seed, OQ.scale_c(p.phi), cache=4)
    total = 0
    for b in range(B):
        xi, xv, recs = OI.qniht_adaptive(p.phi, Y[b], p.s, p.n_iter, p.b_phi, p.b_y, p.seed, p.K, pool=opool,
                                         snapshot=b, mu_fallback=p.mu)
        checked, _ = _compare(recs, idx[:, b].numpy(), val[:, b].numpy(), nnz[:, b].numpy(), mu[:, b].numpy(),
                              sh[:, b].numpy(), 1e-3, 1e-3, 1e-3, 1e-3)
        total += checked
    assert total >= B * 2
    sol.close()


def test_adaptive_rejects_bad_parameters():
    p = CASES["gauss4bit"]()
    pool = _pool(p.phi, p.b_phi, 2, p.seed)
    with pytest.raises(Exception):
        iht.Solver(pool, p.s, 3, p.mu, p.b_y, p.seed, adaptive=True, c=1e-3, k=1.0)   # k <= 1/(1-c)
