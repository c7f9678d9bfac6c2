"""QNIHT oracle in float64 -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows, step by step and in the paper's order:
  * Eq. modified_update_rule / Eq. (3):
        x^{n+1} = H_s( x^n + mu Q(Phi)^dagger ( Q(y) - Q(Phi) x^n ) )
  * Algorithm 1 "QNIHT", lines P:345-351 with a FIXED step mu
    (north star / BASELINE config 1 "step mu=1"; reading c9), independent
    quantised copies Phi-hat_1 .. Phi-hat_{2n*} used as
    g^{[n]} = Phi-hat_{2n-1}^dagger (y-hat - Phi-hat_{2n} x^{[n]})
    with the K-pool reading c6: adjoint copy (2n-2) mod K, forward copy
    (2n-1) mod K (0-based copy ids; K = 2 n* is Algorithm 1 exactly).
  * x^{[1]} = x^{[0]} = 0 (reading c8), so g^{[1]} = Phi-hat_1^dagger y-hat.
  * x is real (x in R^N) and the descent direction is the real part
    Re(Phi-hat^H r) (reading c13).
  * H_s keeps the s largest magnitudes; ties go to the lowest
    index and zeros are never kept (reading c15).

Products are the plain dense definitions: the forward product is "a matrix times
a sparse vector", i.e. Phi-hat[:, S] @ x_S, and the adjoint is
Re(conj(Phi-hat).T @ r).  Everything is float64 (complex128 for the
radio matrices); quantised codes come from oracle.quantize.
"""
from dataclasses import dataclass, field

import numpy as np

from . import quantize as Q


def hard_threshold(a, s):
    """H_s: indices (strictly increasing) and values of the s entries of
    largest |a_i|; ties broken toward the lower index; zero entries never kept
    (so fewer than s are returned when a has fewer than s nonzeros)."""
    a = np.asarray(a, dtype=np.float64)
    if not np.all(np.isfinite(a)):
        raise ValueError("H_s domain error: non-finite input (S:52)")
    if s <= 0:
        return np.zeros(0, dtype=np.int64), np.zeros(0)
    mag = np.abs(a)
    # stable sort on -|a| keeps equal magnitudes in increasing index order
    order = np.argsort(-mag, kind="stable")
    keep = order[:s]
    keep = keep[mag[keep] > 0.0]
    keep = np.sort(keep)
    return keep.astype(np.int64), a[keep]


def forward(phi_hat, x_idx, x_val, y_hat):
    """r = y-hat - Phi-hat x for sparse x."""
    if len(x_idx) == 0:
        return np.array(y_hat, copy=True)
    return y_hat - phi_hat[:, x_idx] @ np.asarray(x_val, dtype=np.float64)


def adjoint(phi_hat, r):
    """g = Re(Phi-hat^H r) (real part per reading c13)."""
    if np.iscomplexobj(phi_hat):
        return np.real(np.conj(phi_hat).T @ r)
    return phi_hat.T @ r


def margin_at_s(a, s):
    """|a|_(s) - |a|_(s+1): gap between the s-th and (s+1)-th largest magnitudes
    (used by the parity rule to flag near-ties; not part of the method)."""
    mag = np.sort(np.abs(a))[::-1]
    if s <= 0 or s >= mag.size:
        return np.inf
    return mag[s - 1] - mag[s]


@dataclass
class IterRecord:
    n: int
    adj_copy: int
    fwd_copy: int
    r: np.ndarray
    g: np.ndarray
    a: np.ndarray
    x_idx: np.ndarray
    x_val: np.ndarray
    margin: float


@dataclass
class QnihtResult:
    x_idx: np.ndarray
    x_val: np.ndarray
    y_hat: np.ndarray
    c_phi: float
    c_y: float
    trace: list = field(default_factory=list)


class CopyPool:
    """The set of independent quantised copies {Phi-hat_k} (Alg. 1 input),
    generated on demand from the counter-based quantizer and cached."""

    def __init__(self, phi, bits, level_mode, seed, c_phi, cache=4):
        self.phi = phi
        self.bits = bits
        self.level_mode = level_mode
        self.seed = seed
        self.c = c_phi
        self.cache = cache
        self._store = {}

    def codes(self, copy_id):
        codes, _ = Q.quantize_matrix(self.phi, self.bits, self.level_mode, self.seed,
                                     copy_id, c=self.c)
        return codes

    def dequantized(self, copy_id):
        if copy_id not in self._store:
            if len(self._store) >= self.cache:
                self._store.pop(next(iter(self._store)))
            self._store[copy_id] = Q.dequantize(self.codes(copy_id), self.c, self.bits,
                                                self.level_mode)
        return self._store[copy_id]


def qniht(phi, y, s, n_iter, mu, b_phi, b_y, seed, K, level_mode=0, record=True,
          x0=None, pool=None, snapshot=0, iter_hook=None):
    """Algorithm 1 with fixed step mu; returns QnihtResult.

    phi: float32 (M x N) or complex64 array; y: float32 / complex64 (M,).
    K: number of independent copies in the pool (reading c6).
    pool: optional pre-built CopyPool of the same (phi, b_phi, seed) -- lets a caller
    time the iterations without the one-time quantisation of the copies.
    snapshot: index b of this observation among B sharing Phi (config 5); selects the
    Philox column of its y-hat (oracle.quantize.quantize_vector).
    iter_hook: optional callable iter_hook(n) invoked after iteration n (timing
    instrumentation for bench.py's CPU baseline; it sees nothing and changes nothing).
    """
    c_phi = Q.scale_c(phi)
    c_y = Q.scale_c(y)
    y_codes, _ = Q.quantize_vector(y, b_y, level_mode, seed, c=c_y, snapshot=snapshot)
    y_hat = Q.dequantize(y_codes, c_y, b_y, level_mode)          # quantised once
    if pool is None:
        pool = CopyPool(phi, b_phi, level_mode, seed, c_phi, cache=max(2, min(K, 4)))
    N = phi.shape[1]
    if x0 is None:
        x_idx, x_val = np.zeros(0, dtype=np.int64), np.zeros(0)  # x^[0] = 0
    else:
        x_idx, x_val = x0
    res = QnihtResult(x_idx, x_val, y_hat, float(c_phi), float(c_y))
    for n in range(1, n_iter + 1):
        a_id = (2 * n - 2) % K          # Phi-hat_{2n-1} (1-based) -> adjoint
        f_id = (2 * n - 1) % K          # Phi-hat_{2n}   (1-based) -> forward
        r = forward(pool.dequantized(f_id), x_idx, x_val, y_hat)
        g = adjoint(pool.dequantized(a_id), r)
        a = np.zeros(N)
        a[x_idx] = x_val
        a = a + mu * g                   # x^[n] + mu g^[n]
        x_idx, x_val = hard_threshold(a, s)
        if record:
            res.trace.append(IterRecord(n, a_id, f_id, r, g, a, x_idx, x_val,
                                        margin_at_s(a, s)))
        if iter_hook is not None:
            iter_hook(n)
    res.x_idx, res.x_val = x_idx, x_val
    return res


def qniht_batched(phi, Y, s, n_iter, mu, b_phi, b_y, seed, K, level_mode=0, record=True):
    """B independent observations sharing one Phi (BASELINE config 5): Algorithm 1 run
    on each column y_b of Y (M x B) with the SAME pool of quantised copies (P:345, P:349
    applied per snapshot); each snapshot has its own c_y and y-hat (snapshot b).  Returns
    a list of QnihtResult."""
    Y = np.asarray(Y)
    c_phi = Q.scale_c(phi)
    pool = CopyPool(phi, b_phi, level_mode, seed, c_phi, cache=max(2, min(K, 4)))
    return [qniht(phi, Y[:, b], s, n_iter, mu, b_phi, b_y, seed, K, level_mode=level_mode, record=record,
                  pool=pool, snapshot=b) for b in range(Y.shape[1])]


def adaptive_step(g, A, gamma):
    """Eq. step_size / Algorithm 1 line 4: mu = (g_G^T g_G) /
    (g_G^T A_G^H A_G g_G) on the support G, with A the quantised copy that produced g
    (reading c10).  Returns None for a zero denominator (degenerate step)."""
    gamma = np.asarray(gamma, dtype=np.int64)
    gg = np.asarray(g, dtype=np.float64)[gamma]
    num = float(gg @ gg)
    Ag = A[:, gamma] @ gg
    den = float(np.real(np.vdot(Ag, Ag)))
    if den == 0.0:
        return None
    return num / den


@dataclass
class AdaptiveRecord:
    n: int
    mu: float
    shrinks: int
    support_changed: bool
    x_idx: np.ndarray
    x_val: np.ndarray
    accept_margin: float = np.inf   # min |mu - (1-c) b| / mu over the acceptance tests (parity rule)
    select_margin: float = np.inf   # |a|_(s) - |a|_(s+1) of the accepted proposal, relative to |a|_(s)


def qniht_adaptive(phi, y, s, n_iter, b_phi, b_y, seed, K, c=1e-3, k=2.0, level_mode=0, max_shrink=60,
                   mu_fallback=1.0, pool=None, snapshot=0, quantized=True):
    """Algorithm 1 "QNIHT" with the adaptive step and the acceptance / shrink
    loop, in the paper's order:

      Gamma^[1] = supp(H_s(Phi-hat_1^H y-hat))
      for n = 1..n*:
        g   = Re(Phi-hat_{2n-1}^H (y-hat - Phi-hat_{2n} x))
        mu  = |g_G|^2 / |Phi-hat_{2n-1}[:, G] g_G|^2, G = Gamma^[n]      (reading c10)
        x'  = H_s(x + mu g), Gamma' = supp(x')
        if Gamma' != Gamma^[n]:                                           (reading c11)
          b = |x' - x|^2 / |Phi-hat_{2n-1}(x' - x)|^2
          while mu > (1 - c) b:  mu <- mu / (k (1 - c));  x' = H_s(x + mu g);  b from the new x'
        x^[n+1] = x', Gamma^[n+1] = supp(x')
    Reading c11: the garbled "x^[n+1] = x^[n]" branches are read as ACCEPT (support unchanged,
    or mu <= (1-c) b), REJECT-and-shrink otherwise.  A zero step denominator falls back to
    mu_fallback.  quantized=False runs the same loop on Phi and y themselves (NIHT).
    Returns (x_idx, x_val, records)."""
    if quantized:
        c_phi = Q.scale_c(phi)
        c_y = Q.scale_c(y)
        y_codes, _ = Q.quantize_vector(y, b_y, level_mode, seed, c=c_y, snapshot=snapshot)
        y_hat = Q.dequantize(y_codes, c_y, b_y, level_mode)
        if pool is None:
            pool = CopyPool(phi, b_phi, level_mode, seed, c_phi, cache=max(2, min(K, 4)))
        mat = pool.dequantized
    else:
        cplx = np.iscomplexobj(phi)
        full = np.asarray(phi, dtype=np.complex128 if cplx else np.float64)
        y_hat = np.asarray(y, dtype=full.dtype)
        mat = lambda _k: full   # noqa: E731
    N = phi.shape[1]
    x_idx, x_val = np.zeros(0, dtype=np.int64), np.zeros(0)
    A1 = mat(0)
    gamma, _ = hard_threshold(adjoint(A1, y_hat), s)                  # Gamma^[1]
    recs = []
    for n in range(1, n_iter + 1):
        A = mat((2 * n - 2) % K)
        F = mat((2 * n - 1) % K)
        g = adjoint(A, forward(F, x_idx, x_val, y_hat))
        mu = adaptive_step(g, A, gamma) if len(gamma) else None
        if mu is None:
            mu = mu_fallback
        xd = np.zeros(N)
        xd[x_idx] = x_val

        def propose(m):
            return hard_threshold(xd + m * g, s)

        ni, nv = propose(mu)
        shrinks = 0
        acc_margin = np.inf
        changed = ni.tolist() != list(gamma)
        if changed:
            while True:
                dx = np.zeros(N)
                dx[ni] = nv
                dx = dx - xd
                sup = np.flatnonzero(dx)
                num = float(dx[sup] @ dx[sup])
                Adx = A[:, sup] @ dx[sup]
                den = float(np.real(np.vdot(Adx, Adx)))
                if num > 0.0 and den > 0.0:
                    acc_margin = min(acc_margin, abs(mu - (1.0 - c) * (num / den)) / mu)
                if num == 0.0 or den == 0.0 or mu <= (1.0 - c) * (num / den):
                    break
                if shrinks >= max_shrink:
                    raise RuntimeError("shrink loop did not terminate")
                mu = mu / (k * (1.0 - c))
                shrinks += 1
                ni, nv = propose(mu)
        x_idx, x_val = ni, nv
        gamma = x_idx
        a = xd + mu * g
        mag = np.sort(np.abs(a))[::-1]
        sel = (mag[s - 1] - mag[s]) / max(mag[s - 1], 1e-300) if 0 < s < N else np.inf
        recs.append(AdaptiveRecord(n, mu, shrinks, changed, x_idx, x_val, acc_margin, sel))
    return x_idx, x_val, recs


def niht_fixed_full_precision(phi, y, s, n_iter, mu):
    """Full-precision IHT with fixed step (Eq. iht_update_rule); exists
    only for the oracle's own pins (b = infinity, no Q)."""
    phi = np.asarray(phi, dtype=np.complex128 if np.iscomplexobj(phi) else np.float64)
    y = np.asarray(y, dtype=phi.dtype)
    N = phi.shape[1]
    x_idx, x_val = np.zeros(0, dtype=np.int64), np.zeros(0)
    for _ in range(n_iter):
        r = forward(phi, x_idx, x_val, y)
        g = adjoint(phi, r)
        a = np.zeros(N)
        a[x_idx] = x_val
        a = a + mu * g
        x_idx, x_val = hard_threshold(a, s)
    return x_idx, x_val


def objective(phi, y, x_idx, x_val):
    """||y - Phi x||_2^2 (Eq. cost_function)."""
    r = forward(np.asarray(phi, dtype=np.complex128), x_idx, x_val,
                np.asarray(y, dtype=np.complex128))
    return float(np.real(np.vdot(r, r)))
