"""Pins for oracle/iht.py: brute force, closed forms and properties the paper fixes.

H_s against brute force over all supports; products against dense
algebra and the adjoint identity; the IHT loop against brute-force l0 (Eq.
cost_function), exact noiseless recovery, the identity matrix,
monotone descent under mu ||Phi-hat||^2 < 1, the unbiased product of
independent copies (proof notation Q_1/Q_2) and b -> large.
"""
import itertools

import numpy as np
import pytest

from oracle import iht as I
from oracle import quantize as Q

SEED = 0xC0FFEE


# ---------------------------------------------------------------- H_s
def test_hard_threshold_spec_examples():
    idx, val = I.hard_threshold([3.0, -5.0, 1.0], 2)
    assert idx.tolist() == [0, 1] and val.tolist() == [3.0, -5.0]
    idx, val = I.hard_threshold([3.0, -3.0, 1.0], 1)           # S:55 tie -> lower index
    assert idx.tolist() == [0] and val.tolist() == [3.0]
    idx, _ = I.hard_threshold([1.0, 2.0], 0)
    assert idx.size == 0


def test_hard_threshold_zeros_and_domain():
    idx, val = I.hard_threshold([0.0, 2.0, 0.0, -1.0], 3)       # fewer nonzeros than s
    assert idx.tolist() == [1, 3]
    with pytest.raises(ValueError):
        I.hard_threshold([1.0, np.nan], 1)
    idx, _ = I.hard_threshold([2.0, -2.0, 2.0, 1.0, -2.0], 3)   # ties resolved by index
    assert idx.tolist() == [0, 1, 2]


def test_hard_threshold_brute_force():
    """||H_s(v) - v|| <= ||w - v|| for every s-sparse w, N <= 8, s <= 3;
    among optimal supports H_s picks the lexicographically lowest."""
    rng = np.random.default_rng(0)
    for trial in range(300):
        N = int(rng.integers(1, 9))
        v = rng.integers(-3, 4, size=N).astype(float) if trial % 2 else rng.standard_normal(N)
        for s in range(0, 4):
            idx, val = I.hard_threshold(v, s)
            h = np.zeros(N)
            h[idx] = val
            best = np.inf
            best_sup = None
            for k in range(0, min(s, N) + 1):
                for sup in itertools.combinations(range(N), k):
                    w = np.zeros(N)
                    w[list(sup)] = v[list(sup)]
                    err = np.linalg.norm(w - v)
                    if err < best - 1e-15:
                        best, best_sup = err, sup
            assert np.linalg.norm(h - v) <= best + 1e-12
            assert len(idx) <= s and np.all(np.diff(idx) > 0)
            # idempotence
            idx2, val2 = I.hard_threshold(h, s)
            assert idx2.tolist() == idx.tolist() and np.array_equal(val2, val)


# ---------------------------------------------------------------- products
def test_forward_adjoint_dense_and_identity():
    rng = np.random.default_rng(1)
    phi = rng.standard_normal((6, 9)) + 1j * rng.standard_normal((6, 9))
    x_idx = np.array([1, 4, 7])
    x_val = rng.standard_normal(3)
    y = rng.standard_normal(6) + 1j * rng.standard_normal(6)
    x = np.zeros(9)
    x[x_idx] = x_val
    np.testing.assert_allclose(I.forward(phi, x_idx, x_val, y), y - phi @ x, rtol=1e-13)
    r = rng.standard_normal(6) + 1j * rng.standard_normal(6)
    g = I.adjoint(phi, r)
    # Re<Phi x, r> = <x, Re(Phi^H r)> for real x
    xr = rng.standard_normal(9)
    lhs = np.real(np.vdot(r, phi @ xr))
    assert abs(lhs - xr @ g) <= 1e-10 * abs(lhs)
    # scalar loop definition: g_n = Re sum_m conj(Phi_mn) r_m
    loop = [sum((np.conj(phi[m, n]) * r[m]).real for m in range(6)) for n in range(9)]
    np.testing.assert_allclose(g, loop, rtol=1e-12)
    assert I.adjoint(np.array([[1j]]), np.array([1.0]))[0] == 0.0


# ---------------------------------------------------------------- loop
def _l0_brute(phi, y, s):
    best = (np.inf, None, None)
    for sup in itertools.combinations(range(phi.shape[1]), s):
        sup = list(sup)
        xs, *_ = np.linalg.lstsq(phi[:, sup], y, rcond=None)
        o = np.sum((y - phi[:, sup] @ xs) ** 2)
        if o < best[0]:
            best = (o, sup, xs)
    return best


def test_iht_against_bruteforce_l0():
    """M=8, N=16, s=2, noiseless Gaussian; mu = 1/||Phi||^2 (descent guaranteed,
    P:209).  The brute-force l0 minimum never exceeds the IHT objective;
    when IHT finds the optimal support its values are the least-squares ones."""
    agree = 0
    for seed in range(40):
        rng = np.random.default_rng(seed)
        M, N, s = 8, 16, 2
        phi = rng.standard_normal((M, N))
        x = np.zeros(N)
        S = rng.choice(N, s, replace=False)
        x[S] = rng.standard_normal(s)
        y = phi @ x
        best_obj, best_sup, best_x = _l0_brute(phi, y, s)
        mu = 1.0 / np.linalg.norm(phi, 2) ** 2
        xi, xv = I.niht_fixed_full_precision(phi, y, s, 3000, mu)
        obj = I.objective(phi, y, xi, xv)
        assert best_obj <= obj + 1e-12
        if list(xi) == best_sup:
            agree += 1
            np.testing.assert_allclose(xv, best_x, rtol=1e-6, atol=1e-9)
    assert agree >= 10, agree


@pytest.mark.parametrize("M,N,s", [(256, 512, 8), (256, 1024, 16)])
def test_exact_noiseless_recovery_full_precision(M, N, s):
    """Gaussian N(0,1/M) Phi, +-1 spikes, noiseless, mu = 1: exact recovery."""
    for seed in range(3):
        rng = np.random.default_rng(10 + seed)
        phi = rng.standard_normal((M, N)) / np.sqrt(M)
        x = np.zeros(N)
        S = rng.choice(N, s, replace=False)
        x[S] = rng.choice([-1.0, 1.0], s)
        xi, xv = I.niht_fixed_full_precision(phi, phi @ x, s, 300, 1.0)
        xr = np.zeros(N)
        xr[xi] = xv
        assert np.linalg.norm(xr - x) / np.linalg.norm(x) < 1e-6


def test_identity_recovers_in_one_step():
    """Phi = I, noiseless, s = ||x||_0: exact after one iteration."""
    x = np.zeros(12)
    x[[2, 5, 9]] = [1.5, -2.0, 0.25]
    xi, xv = I.niht_fixed_full_precision(np.eye(12), x, 3, 1, 1.0)
    assert xi.tolist() == [2, 5, 9] and np.allclose(xv, [1.5, -2.0, 0.25])


def test_monotone_descent_single_copy():
    """With one fixed quantised matrix (K = 1) and mu ||Phi-hat||^2 < 1 the
    majorisation argument of Sec. 3 "Convergence" gives
    ||y-hat - Phi-hat x^{n+1}|| <= ||y-hat - Phi-hat x^n||."""
    rng = np.random.default_rng(5)
    M, N, s = 64, 128, 6
    phi = (rng.standard_normal((M, N)) / np.sqrt(M)).astype(np.float32)
    x = np.zeros(N)
    x[rng.choice(N, s, replace=False)] = rng.standard_normal(s)
    y = (phi.astype(np.float64) @ x + 0.01 * rng.standard_normal(M)).astype(np.float32)
    A = Q.dequantize(Q.quantize_matrix(phi, 4, 0, SEED, 0)[0], Q.scale_c(phi), 4, 0)
    mu = 0.99 / np.linalg.norm(A, 2) ** 2
    res = I.qniht(phi, y, s, 60, mu, 4, 8, SEED, K=1)
    norms = [np.linalg.norm(t.r) for t in res.trace]
    assert all(norms[i + 1] <= norms[i] * (1 + 1e-12) for i in range(len(norms) - 1))


def test_independent_copies_unbiased_product():
    """E[Q_1(Phi)^T Q_2(Phi)] = Phi^T Phi for independent copies,
    while a single copy's Gram matrix is biased on the diagonal by the
    quantisation variance; copies are drawn exactly as the solver draws them."""
    rng = np.random.default_rng(6)
    phi = rng.standard_normal((16, 5)).astype(np.float32)
    c = Q.scale_c(phi)
    P = phi.astype(np.float64)
    acc_ind = np.zeros((5, 5))
    acc_same = np.zeros((5, 5))
    n = 600
    for k in range(n):
        A = Q.dequantize(Q.quantize_matrix(phi, 2, 0, SEED, 2 * k)[0], c, 2, 0)
        F = Q.dequantize(Q.quantize_matrix(phi, 2, 0, SEED, 2 * k + 1)[0], c, 2, 0)
        acc_ind += A.T @ F
        acc_same += A.T @ A
    ref = P.T @ P
    scale = np.abs(ref).max()
    assert np.abs(acc_ind / n - ref).max() < 0.08 * scale
    assert np.min(np.diag(acc_same / n - ref)) > 0.1 * scale     # biased upwards


def test_large_bits_approach_full_precision():
    """b_Phi = b_y = 16: QNIHT agrees with full-precision IHT within 1e-3."""
    rng = np.random.default_rng(7)
    M, N, s = 128, 256, 5
    phi = (rng.standard_normal((M, N)) / np.sqrt(M)).astype(np.float32)
    x = np.zeros(N)
    x[rng.choice(N, s, replace=False)] = rng.choice([-1.0, 1.0], s)
    y = (phi.astype(np.float64) @ x).astype(np.float32)
    xi0, xv0 = I.niht_fixed_full_precision(phi, y, s, 100, 1.0)
    res = I.qniht(phi, y, s, 100, 1.0, 16, 16, SEED, K=200, record=False)
    assert res.x_idx.tolist() == xi0.tolist()
    assert np.linalg.norm(res.x_val - xv0) / np.linalg.norm(xv0) < 1e-3


def test_row_sharded_adjoint_sums_to_full():
    """Row sharding (north star, 8(e)): sum of per-shard adjoints = full adjoint."""
    rng = np.random.default_rng(8)
    A = rng.standard_normal((40, 11)) + 1j * rng.standard_normal((40, 11))
    r = rng.standard_normal(40) + 1j * rng.standard_normal(40)
    parts = sum(I.adjoint(A[a:b], r[a:b]) for a, b in [(0, 13), (13, 29), (29, 40)])
    np.testing.assert_allclose(parts, I.adjoint(A, r), rtol=1e-12)


def _identify_copy(copies, vec_in, out, op):
    """Which of the candidate dequantised copies reproduces `out` = op(copy, vec_in)?"""
    hits = [k for k, D in enumerate(copies) if np.allclose(op(D, vec_in), out, rtol=1e-12, atol=1e-12)]
    return hits


@pytest.mark.parametrize("K", [2, 6])
def test_copy_roles_follow_algorithm1(K):
    """Pin of the copy-role map (readings c6-c8; Algorithm 1).  With strongly
    distinct 2-bit copies, each iteration's recorded r and g are matched by brute force
    against EVERY copy of the pool (each dequantised from oracle.quantize, the pinned
    quantiser), independently of qniht's own bookkeeping:
      * iteration 1's gradient is Phi-hat_1^dagger y-hat with Phi-hat_1 = copy 0 -- the
        vector whose H_s gives Gamma^1, since x^[1] = 0 (c8);
      * the adjoint of iteration n uses the odd-labelled copy Phi-hat_{2n-1} and the forward
        the even-labelled Phi-hat_{2n} (c7), i.e. 0-based ids (2n-2, 2n-1) mod K;
      * forward and adjoint of one iteration never share a copy (the Q_1 / Q_2 independence
        of the proof), and with K = 2 n* every copy is used exactly once.
    Swapping the roles, or using one copy for both, fails this test."""
    rng = np.random.default_rng(11)
    M, N, s, n_iter = 40, 96, 4, K // 2 if K > 2 else 3
    phi = rng.standard_normal((M, N)).astype(np.float32)
    x = np.zeros(N)
    x[rng.choice(N, s, replace=False)] = rng.standard_normal(s)
    y = (phi.astype(np.float64) @ x).astype(np.float32)
    res = I.qniht(phi, y, s, n_iter, 0.5, 2, 8, SEED, K, record=True)
    c = Q.scale_c(phi)
    copies = [Q.dequantize(Q.quantize_matrix(phi, 2, 0, SEED, k, c=c)[0], c, 2, 0) for k in range(K)]
    for a in range(K):                      # the copies really are distinct at 2 bits
        for b in range(a + 1, K):
            assert np.abs(copies[a] - copies[b]).max() > 0.5 * c
    # iteration 1: g = Phi-hat_1^T y-hat (x^[1] = 0, so r = y-hat), Gamma^1 from it
    assert np.array_equal(res.trace[0].r, res.y_hat)
    assert _identify_copy(copies, res.y_hat, res.trace[0].g, lambda D, v: D.T @ v) == [0]
    g1_idx, _ = I.hard_threshold(copies[0].T @ res.y_hat, s)
    assert res.trace[0].x_idx.tolist() == g1_idx.tolist()        # mu > 0 keeps H_s's support
    used = []
    x_idx, x_val = np.zeros(0, np.int64), np.zeros(0)
    for n, rec in enumerate(res.trace, start=1):
        fwd = _identify_copy(copies, (x_idx, x_val), rec.r,
                             lambda D, xv: res.y_hat - D[:, xv[0]] @ xv[1] if len(xv[0]) else res.y_hat)
        adj = _identify_copy(copies, rec.r, rec.g, lambda D, v: D.T @ v)
        assert adj == [(2 * n - 2) % K], (n, adj)
        if n > 1:                            # at n = 1 x = 0: every copy gives r = y-hat
            assert fwd == [(2 * n - 1) % K], (n, fwd)
            assert fwd != adj
            used.append(fwd[0])
        used.append(adj[0])
        x_idx, x_val = rec.x_idx, rec.x_val
    if K == 2 * n_iter:                      # Algorithm 1 exactly: each copy once (fwd of n=1 unused)
        assert sorted(used) == sorted(set(used)) and len(used) == K - 1
