"""Pins of the adaptive-step oracle (Algorithm 1 with mu-hat, acceptance and shrink;
SURVEY 8(f) NEXT-1) against closed forms and properties the paper fixes.

* adaptive_step: identity -> 1, 2 I -> 1/4 (S:193-195 examples); and mu is the exact
  minimiser of the residual along the support-restricted gradient ("the maximal
  reduction in cost function can then be attained"), checked by perturbing mu.
* NIHT (full precision, same loop): identity recovers in one iteration; Gaussian
  256 x 512, 8-sparse +-1, noiseless: exact recovery on >= 19 of 20 seeds (S:204,
  supp. P:1217); residual never increases across accepted steps (Theorem 1 / S:215).
* QNIHT with 16-bit Phi and y approaches NIHT.
* The shrink loop runs on a case where the first proposal is rejected, and its accepted
  step satisfies mu <= (1 - c) b.
"""
import numpy as np
import pytest

from oracle import iht as OI


def test_adaptive_step_closed_forms():
    rng = np.random.default_rng(1)
    g = rng.standard_normal(12)
    gamma = np.array([1, 4, 7])
    assert OI.adaptive_step(g, np.eye(12), gamma) == pytest.approx(1.0, rel=1e-15)
    assert OI.adaptive_step(g, 2 * np.eye(12), gamma) == pytest.approx(0.25, rel=1e-15)
    assert OI.adaptive_step(np.zeros(12), np.eye(12), gamma) is None      # degenerate: zero denominator


def test_adaptive_step_is_exact_line_search():
    rng = np.random.default_rng(2)
    for trial in range(20):
        A = rng.standard_normal((8, 12))
        r = rng.standard_normal(8)
        g = A.T @ r                                   # gradient at the current iterate
        gamma = np.sort(rng.choice(12, 3, replace=False))
        d = np.zeros(12)
        d[gamma] = g[gamma]
        mu = OI.adaptive_step(g, A, gamma)
        f = lambda t: float(np.sum((r - t * (A @ d)) ** 2))   # noqa: E731
        for eps in (1e-3, 1e-6):
            assert f(mu) <= f(mu * (1 + eps)) and f(mu) <= f(mu * (1 - eps))


def test_niht_identity_one_iteration():
    N, s = 40, 5
    rng = np.random.default_rng(3)
    x = np.zeros(N)
    idx = np.sort(rng.choice(N, s, replace=False))
    x[idx] = rng.standard_normal(s)
    xi, xv, recs = OI.qniht_adaptive(np.eye(N), x, s, 1, 0, 0, 0, 1, quantized=False)
    assert xi.tolist() == idx.tolist()
    np.testing.assert_allclose(xv, x[idx], rtol=0, atol=1e-15)


def _gauss(seed, M=256, N=512, s=8):
    rng = np.random.default_rng(seed)
    phi = rng.standard_normal((M, N)) / np.sqrt(M)
    idx = np.sort(rng.choice(N, s, replace=False))
    x = np.zeros(N)
    x[idx] = rng.choice([-1.0, 1.0], s)
    return phi, x, phi @ x


def test_niht_gaussian_recovery_rate_and_descent():
    ok = 0
    for seed in range(20):
        phi, x, y = _gauss(seed)
        xi, xv, recs = OI.qniht_adaptive(phi, y, 8, 100, 0, 0, 0, 1, quantized=False)
        xr = np.zeros(512)
        xr[xi] = xv
        ok += np.linalg.norm(xr - x) / np.linalg.norm(x) < 1e-4
        # monotone descent over the accepted iterates
        prev = np.linalg.norm(y)
        for rec in recs:
            xd = np.zeros(512)
            xd[rec.x_idx] = rec.x_val
            cur = np.linalg.norm(y - phi @ xd)
            assert cur <= prev + 1e-10
            prev = cur
    assert ok >= 19


def test_shrink_loop_accepts_only_admissible_steps():
    found = False
    for seed in range(40):
        phi, x, y = _gauss(100 + seed, M=64, N=256, s=10)
        phi = phi * 3.0                               # large RIP constants: first proposals overshoot
        xi, xv, recs = OI.qniht_adaptive(phi, y, 10, 15, 0, 0, 0, 1, quantized=False, c=1e-3, k=2.0)
        xprev = np.zeros(256)
        for rec in recs:
            xn = np.zeros(256)
            xn[rec.x_idx] = rec.x_val
            if rec.support_changed:
                dx = xn - xprev
                den = np.sum((phi @ dx) ** 2)
                if den > 0 and np.any(dx):
                    assert rec.mu <= (1 - 1e-3) * np.sum(dx ** 2) / den * (1 + 1e-12)
            found |= rec.shrinks > 0
            xprev = xn
    assert found, "no rejected proposal in the sample: the shrink branch was not exercised"


def test_qniht_adaptive_16bit_approaches_niht():
    phi, x, y = _gauss(7)
    xi0, xv0, _ = OI.qniht_adaptive(phi, y, 8, 30, 0, 0, 0, 1, quantized=False)
    xi1, xv1, _ = OI.qniht_adaptive(phi.astype(np.float32), y.astype(np.float32), 8, 30, 16, 16, 11, 60)
    assert xi0.tolist() == xi1.tolist()
    assert np.linalg.norm(xv1 - xv0) / np.linalg.norm(xv0) < 1e-3
