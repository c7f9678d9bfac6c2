"""GPU parity of the batched path (BASELINE config 5: B observations sharing one Phi),
through the C ABI, against the float64 CPU oracle run per snapshot.

Bar: y-hat codes bit-exact per snapshot; forward within 1e-4 (fp32 CUDA cores); adjoint
within 1e-3 relative l2 (the tensor-core path's tolerance, north star: r enters the int8
MMA in 15-bit block fixed point); H_s exact on identical fp32 inputs; the column-shard
merge identical to the unsharded selection; the batched solver identical in support to
the oracle's per-snapshot trajectories away from near-ties, x within 1e-3.
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
TOL_F = 1e-4          # fp32 CUDA-core kernels
TOL_T = 1e-3          # tensor-core (batched adjoint) path
SEED = 0x1802_0490_7B5


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


# ------------------------------------------------------------------ (a1) (a3) per snapshot
@pytest.mark.parametrize("cplx,bits,B", [(True, 8, 64), (False, 8, 5), (False, 4, 1)])
def test_absmax_and_quantize_vec_batched_bit_exact(cplx, bits, B):
    M = 777
    rng = np.random.default_rng(B)
    Y = rng.standard_normal((B, M)) * rng.uniform(0.1, 10, size=(B, 1))
    if cplx:
        Y = Y + 1j * rng.standard_normal((B, M))
    Y = Y.astype(np.complex64 if cplx else np.float32)
    Yd = _to_dev(Y)
    c = iht.absmax_batched(Yd)
    yhat, codes = iht.quantize_vec_batched(Yd, bits, 0, SEED, c, with_codes=True)
    c, yhat, codes = c.cpu().numpy(), yhat.cpu().numpy(), codes.cpu().numpy()
    for b in range(B):
        ref_codes, cb = OQ.quantize_vector(Y[b], bits, 0, SEED, snapshot=b)
        assert np.float32(c[b]) == cb
        np.testing.assert_array_equal(codes[b].reshape(ref_codes.shape), ref_codes)
        assert rel_l2(yhat[b], stack(OQ.dequantize(ref_codes, cb, bits, 0), M)) < 1e-6
    # snapshot 0 is exactly the single-observation quantiser
    y0, c0 = iht.quantize_vec(_to_dev(Y[0]), bits, 0, SEED, iht.absmax(_to_dev(Y[0])), with_codes=True)
    np.testing.assert_array_equal(c0.cpu().numpy(), codes[0])


# ------------------------------------------------------------------ (a7) batched adjoint
BADJ = [(300, 500, False, 2, 8), (144, 2304, True, 2, 8), (1000, 1000, False, 4, 16), (1000, 700, False, 8, 16),
        (2304, 1500, True, 2, 64), (513, 129, True, 4, 24), (256, 16, False, 2, 8), (300, 500, False, 2, 5),
        (144, 300, True, 2, 72),
        # more tiles than SMs: the last partial wave runs as snapshot halves (N = B columns)
        (256, 22784, False, 2, 16), (100, 24000, True, 8, 48), (100, 24000, True, 4, 40)]


@pytest.mark.parametrize("M,N,cplx,bits,B", BADJ)
def test_adjoint_batched_parity(M, N, cplx, bits, B):
    phi = _phi(M, N, cplx, seed=M + N)
    c = OQ.scale_c(phi)
    (A,) = iht.quantize(_to_dev(phi), bits, 0, SEED, [3], float(c))
    Ad = OQ.dequantize(OQ.quantize_matrix(phi, bits, 0, SEED, 3, c=c)[0], c, bits, 0)
    rng = np.random.default_rng(B)
    planes = 2 if cplx else 1
    R = np.stack([stack(rng.standard_normal(M) + (1j * rng.standard_normal(M) if cplx else 0), M)
                  for _ in range(B)]).astype(np.float32)
    R[1] *= 1e-6                      # per-snapshot scales are independent
    R[2, : M // 5] *= 1e-3            # dynamic range inside one snapshot
    Gm = iht.adjoint_batched(A, _to_dev(R)).cpu().numpy()
    for b in range(B):
        ref = OI.adjoint(Ad, unstack(R[b], M, planes))
        assert rel_l2(Gm[b], ref) < TOL_T, (b, rel_l2(Gm[b], ref))


def test_adjoint_batched_zero_snapshot():
    M, N, B = 512, 300, 8
    phi = _phi(M, N, False, seed=9)
    c = OQ.scale_c(phi)
    (A,) = iht.quantize(_to_dev(phi), 2, 0, SEED, [0], float(c))
    R = torch.zeros((B, iht.vec_len(M, 1)), device=_dev())
    R[3, :M] = torch.randn(M, device=_dev())
    Gm = iht.adjoint_batched(A, R)
    assert torch.count_nonzero(Gm[[0, 1, 2, 4, 5, 6, 7]]) == 0
    assert torch.count_nonzero(Gm[3]) > 0


# ------------------------------------------------------------------ (a4) batched forward
@pytest.mark.parametrize("M,N,cplx,bits,B,s", [(300, 1001, False, 2, 5, 9), (144, 2304, True, 2, 64, 64),
                                                (1000, 700, False, 8, 3, 0),
                                                # > 4 x 148 narrow CTAs: the 32-word-per-CTA layout
                                                (2304, 300, True, 2, 64, 64), (3000, 200, False, 4, 40, 30),
                                                (1100, 150, False, 8, 100, 17)])
def test_forward_batched_parity_and_shards(M, N, cplx, bits, B, s):
    phi = _phi(M, N, cplx, seed=7)
    c = OQ.scale_c(phi)
    (F,) = iht.quantize(_to_dev(phi), bits, 0, SEED, [4], float(c))
    Fd = OQ.dequantize(OQ.quantize_matrix(phi, bits, 0, SEED, 4, c=c)[0], c, bits, 0)
    planes = 2 if cplx else 1
    rng = np.random.default_rng(s)
    ldx = max(s, 1)
    xi = np.zeros((B, ldx), np.int32)
    xv = np.zeros((B, ldx), np.float32)
    nz = np.zeros(B, np.int32)
    for b in range(B):
        k = int(rng.integers(0, s + 1))
        xi[b, :k] = np.sort(rng.choice(N, k, replace=False))
        xv[b, :k] = rng.standard_normal(k)
        nz[b] = k
    Yh = np.stack([stack(rng.standard_normal(M) + (1j * rng.standard_normal(M) if cplx else 0), M)
                   for _ in range(B)]).astype(np.float32)
    Rg = iht.forward_batched(F, _to_dev(xi), _to_dev(xv), _to_dev(nz), _to_dev(Yh)).cpu().numpy()
    for b in range(B):
        k = nz[b]
        ref = OI.forward(Fd, xi[b, :k], xv[b, :k].astype(np.float64), unstack(Yh[b], M, planes))
        assert rel_l2(unstack(Rg[b], M, planes), ref) < TOL_F
    # column shards: partial products over two shards sum to the whole (y-hat on shard 0)
    if N >= 32:
        n0 = (N // 2) // 16 * 16
        parts = []
        for lo, hi, yh in ((0, n0, Yh), (n0, N, None)):
            (Fs,) = iht.quantize(_to_dev(np.ascontiguousarray(phi[:, lo:hi])), bits, 0, SEED, [4], float(c),
                                 col_offset=lo)
            parts.append(iht.forward_batched(Fs, _to_dev(xi), _to_dev(xv), _to_dev(nz),
                                             None if yh is None else _to_dev(yh)).cpu().numpy())
        assert rel_l2(parts[0] + parts[1], Rg) < TOL_F


# ------------------------------------------------------------------ (a6) batched H_s + merge
def _a32(x_idx, x_val, g, mu):
    a = (np.float32(mu) * np.asarray(g, np.float32)).astype(np.float32)
    x_idx = np.asarray(x_idx, np.int64)
    a[x_idx] = (np.asarray(x_val, np.float32) + a[x_idx]).astype(np.float32)
    return a


@pytest.mark.parametrize("N,s,B", [(65536, 64, 64), (1001, 37, 3), (5000, 0, 2), (300, 400, 4)])
def test_threshold_batched_exact_and_merge(N, s, B):
    rng = np.random.default_rng(N + s + B)
    Gm = rng.standard_normal((B, N)).astype(np.float32)
    Gm[1 % B, ::7] = 0.25                                   # ties
    ldx = max(s, 1)
    xi = np.zeros((B, ldx), np.int32)
    xv = np.zeros((B, ldx), np.float32)
    nz = np.zeros(B, np.int32)
    for b in range(B):
        k = min(s, N)
        xi[b, :k] = np.sort(rng.choice(N, k, replace=False))
        xv[b, :k] = rng.standard_normal(k)
        nz[b] = k
    mu = 0.37
    oi, ov, on = iht.threshold_batched(_to_dev(xi), _to_dev(xv), _to_dev(nz), _to_dev(Gm), mu, s)
    oi, ov, on = oi.cpu().numpy(), ov.cpu().numpy(), on.cpu().numpy()
    for b in range(B):
        a = _a32(xi[b, :nz[b]], xv[b, :nz[b]], Gm[b], mu)
        ri, rv = OI.hard_threshold(a.astype(np.float64), s)
        assert oi[b, :on[b]].tolist() == ri.tolist()
        np.testing.assert_array_equal(ov[b, :on[b]], rv.astype(np.float32))
    # column shards (P = 3, widths multiple of 16): local candidates + merge = global H_s
    if s > 0 and N >= 64:
        cuts = [0, (N // 3) // 16 * 16, (2 * N // 3) // 16 * 16, N]
        ci, cv, cn = [], [], []
        for lo, hi in zip(cuts[:-1], cuts[1:]):
            li, lv, ln = iht.threshold_batched(_to_dev(xi), _to_dev(xv), _to_dev(nz),
                                               _to_dev(np.ascontiguousarray(Gm[:, lo:hi])), mu, s, col_offset=lo)
            ci.append(li)
            cv.append(lv)
            cn.append(ln)
        mi, mv, mn = iht.merge_candidates(torch.stack(ci), torch.stack(cv), torch.stack(cn), s)
        mi, mv, mn = mi.cpu().numpy(), mv.cpu().numpy(), mn.cpu().numpy()
        np.testing.assert_array_equal(mn, on)
        for b in range(B):
            assert mi[b, :mn[b]].tolist() == oi[b, :on[b]].tolist()
            np.testing.assert_array_equal(mv[b, :mn[b]], ov[b, :on[b]])


def test_threshold_batched_nan_isolated_to_snapshot():
    Gm = np.ones((3, 1000), np.float32)
    Gm[1, 10] = np.nan
    z = torch.zeros((3, 4), dtype=torch.int32, device=_dev())
    oi, ov, on = iht.threshold_batched(z, z.float(), torch.zeros(3, dtype=torch.int32, device=_dev()),
                                       _to_dev(Gm), 1.0, 4)
    assert on.cpu().numpy().tolist() == [4, -1, 4]


# ------------------------------------------------------------------ solver (batched)
def _radio_batch(B, cfg_id=51, A=12, grid=48, n_src=8, n_iter=20, K=40, b_phi=2):
    p = G.radio_problem(cfg_id=cfg_id, A=A, grid=grid, n_src=n_src, n_iter=n_iter, K=K, b_phi=b_phi, batch=B)
    return p, np.ascontiguousarray(p.meta["batch_y"].T)          # (B, M)


def _near_tie(rec, s, rel):
    a = np.sort(np.abs(rec.a))[::-1]
    kth = a[min(s, a.size) - 1] if s > 0 else 0.0
    return rec.margin <= rel * max(kth, 1e-30)


@pytest.mark.parametrize("B,b_phi", [(16, 2), (5, 4), (72, 2)])
def test_batched_teacher_forced(B, b_phi):
    """Per snapshot and iteration, feed the oracle's x^[n] (and r) into the batched kernels."""
    p, Y = _radio_batch(B, b_phi=b_phi, n_iter=8, K=16)
    refs = OI.qniht_batched(p.phi, Y.T, p.s, p.n_iter, p.mu, p.b_phi, p.b_y, p.seed, p.K)
    pool = iht.quantize(_to_dev(p.phi), p.b_phi, 0, p.seed, list(range(p.K)), float(OQ.scale_c(p.phi)))
    Yd = _to_dev(Y)
    yhat, _ = iht.quantize_vec_batched(Yd, p.b_y, 0, p.seed, iht.absmax_batched(Yd))
    for b in range(B):
        assert rel_l2(yhat[b].cpu().numpy(), stack(refs[b].y_hat, p.M)) < 1e-6
    s, ldx = p.s, p.s
    xi = np.zeros((B, ldx), np.int32)
    xv = np.zeros((B, ldx), np.float32)
    nz = np.zeros(B, np.int32)
    for n in range(p.n_iter):
        recs = [refs[b].trace[n] for b in range(B)]
        Rg = iht.forward_batched(pool[recs[0].fwd_copy], _to_dev(xi), _to_dev(xv), _to_dev(nz), yhat).cpu().numpy()
        R_or = np.stack([stack(r.r, p.M) for r in recs]).astype(np.float32)
        Gm = iht.adjoint_batched(pool[recs[0].adj_copy], _to_dev(R_or)).cpu().numpy()
        g_or = np.stack([r.g for r in recs]).astype(np.float32)
        oi, ov, on = iht.threshold_batched(_to_dev(xi), _to_dev(xv), _to_dev(nz), _to_dev(g_or), p.mu, s)
        oi, ov, on = oi.cpu().numpy(), ov.cpu().numpy(), on.cpu().numpy()
        for b, rec in enumerate(recs):
            assert rel_l2(unstack(Rg[b], p.M, 2), rec.r) < TOL_F, (n, b)
            assert rel_l2(Gm[b], rec.g) < TOL_T, (n, b)
            if not _near_tie(rec, s, 1e-5):
                assert oi[b, :on[b]].tolist() == rec.x_idx.tolist(), (n, b)
                assert rel_l2(ov[b, :on[b]], rec.x_val, floor=1e-30) < TOL_F
            k = len(rec.x_idx)
            xi[b] = 0
            xv[b] = 0
            xi[b, :k] = rec.x_idx
            xv[b, :k] = rec.x_val
            nz[b] = k


@pytest.mark.parametrize("B,graph", [(16, True), (16, False), (64, True)])
def test_batched_solver_free_running(B, graph):
    p, Y = _radio_batch(B, n_iter=20, K=40)
    refs = OI.qniht_batched(p.phi, Y.T, p.s, p.n_iter, p.mu, p.b_phi, p.b_y, p.seed, p.K)
    pool = iht.quantize(_to_dev(p.phi), p.b_phi, 0, p.seed, list(range(p.K)), float(OQ.scale_c(p.phi)))
    sol = iht.Solver(pool, p.s, p.n_iter, p.mu, p.b_y, p.seed, trace=True, use_graph=graph, nrhs=B)
    fi, fv, fn = sol.run(_to_dev(Y))
    torch.cuda.synchronize()
    fi, fv, fn = fi.cpu().numpy(), fv.cpu().numpy(), fn.cpu().numpy()
    idx, val, nnz = sol.trace_arrays()
    clean_snapshots = checked = 0
    for b in range(B):
        clean = True
        for n, rec in enumerate(refs[b].trace):
            # the tensor-core adjoint carries ~1e-4 relative error: near-ties at that level may flip,
            # after which the trajectories legitimately part
            if _near_tie(rec, p.s, 1e-3):
                clean = False
                break
            k = int(nnz[n, b])
            assert idx[n, b, :k].numpy().tolist() == rec.x_idx.tolist(), (b, n)
            assert rel_l2(val[n, b, :k].numpy(), rec.x_val, floor=1e-30) < TOL_T, (b, n)
            checked += 1
        if clean:
            clean_snapshots += 1
            assert fi[b, :fn[b]].tolist() == refs[b].x_idx.tolist()
    # never vacuous: most snapshots run clean to the end, and at least 3/4 of all
    # snapshot-iterations are compared
    assert clean_snapshots >= B // 2 and checked >= 3 * B * p.n_iter // 4, (clean_snapshots, checked)
    # deterministic replay
    gi, gv, gn = sol.run(_to_dev(Y))
    torch.cuda.synchronize()
    assert np.array_equal(gi.cpu().numpy(), fi) and np.array_equal(gv.cpu().numpy(), fv)
    sol.close()


def test_batched_solver_host_io():
    B = 8
    p, Y = _radio_batch(B, n_iter=6, K=12)
    pool = iht.quantize(_to_dev(p.phi), p.b_phi, 0, p.seed, list(range(p.K)), float(OQ.scale_c(p.phi)))
    sol = iht.Solver(pool, p.s, p.n_iter, p.mu, p.b_y, p.seed, nrhs=B)
    di, dv, dn = sol.run(_to_dev(Y))
    torch.cuda.synchronize()
    di, dv, dn = di.cpu().clone(), dv.cpu().clone(), dn.cpu().clone()
    yh = torch.from_numpy(Y).pin_memory()
    oi = torch.empty((B, p.s), dtype=torch.int32).pin_memory()
    ov = torch.empty((B, p.s), dtype=torch.float32).pin_memory()
    on = torch.empty(B, dtype=torch.int32).pin_memory()
    sol.run_host(yh, oi, ov, on)
    assert torch.equal(oi, di) and torch.equal(ov, dv) and torch.equal(on, dn)
    sol.close()


def test_batched_solver_world1_column_shard_path():
    """The column-sharded code path (forward partials all-reduced, candidates all-gathered and
    merged) at world size 1 through NCCL gives bit-identical results to the plain batched run."""
    B = 8
    p, Y = _radio_batch(B, n_iter=6, K=12)
    pool = iht.quantize(_to_dev(p.phi), p.b_phi, 0, p.seed, list(range(p.K)), float(OQ.scale_c(p.phi)))
    ref = iht.Solver(pool, p.s, p.n_iter, p.mu, p.b_y, p.seed, nrhs=B)
    ri, rv, rn = [t.cpu().clone() for t in ref.run(_to_dev(Y))]
    comm = iht.Comm(0, 1, 0)
    try:
        sol = iht.Solver(pool, p.s, p.n_iter, p.mu, p.b_y, p.seed, nrhs=B, comm=comm)
        gi, gv, gn = sol.run(_to_dev(Y))
        torch.cuda.synchronize()
        assert torch.equal(gi.cpu(), ri) and torch.equal(gv.cpu(), rv) and torch.equal(gn.cpu(), rn)
        sol.close()
    finally:
        comm.close()
    ref.close()


@pytest.mark.parametrize("bits", [2, 4, 8])
def test_adjoint_batched_odd_level_mode(bits):
    """Odd level mode (2^{b-1}+1 levels, exact zero) on the tcgen05 path."""
    M, N, B = 700, 333, 16
    phi = _phi(M, N, True, seed=bits)
    c = OQ.scale_c(phi)
    (A,) = iht.quantize(_to_dev(phi), bits, 1, SEED, [9], float(c))
    Ad = OQ.dequantize(OQ.quantize_matrix(phi, bits, 1, SEED, 9, c=c)[0], c, bits, 1)
    rng = np.random.default_rng(bits)
    R = np.stack([stack(rng.standard_normal(M) + 1j * rng.standard_normal(M), M) for _ in range(B)]).astype(np.float32)
    Gm = iht.adjoint_batched(A, _to_dev(R)).cpu().numpy()
    for b in range(B):
        assert rel_l2(Gm[b], OI.adjoint(Ad, unstack(R[b], M, 2))) < TOL_T


def test_batched_solver_nan_snapshot_isolated():
    """A non-finite observation poisons only its own snapshot (out_nnz = -1); the others
    are unaffected and equal the run without it."""
    B = 8
    p, Y = _radio_batch(B, n_iter=5, K=10)
    pool = iht.quantize(_to_dev(p.phi), p.b_phi, 0, p.seed, list(range(p.K)), float(OQ.scale_c(p.phi)))
    sol = iht.Solver(pool, p.s, p.n_iter, p.mu, p.b_y, p.seed, nrhs=B)
    ri, rv, rn = [t.cpu().clone() for t in sol.run(_to_dev(Y))]
    Y2 = Y.copy()
    Y2[5, 7] = np.nan
    gi, gv, gn = [t.cpu().clone() for t in sol.run(_to_dev(Y2))]
    assert int(gn[5]) == -1
    keep = [b for b in range(B) if b != 5]
    assert torch.equal(gn[keep], rn[keep]) and torch.equal(gi[keep], ri[keep]) and torch.equal(gv[keep], rv[keep])
    sol.close()


# ------------------------------------------------------------------ bounded select (config 5)
def _bounded_runs(pool, p, Y, B, n_iter, monkeypatch, capfd, bound="0.5"):
    """The batched solver's trace with the bounded select off and on (IHT_BOUNDED, read at
    every create), and the on-run's decided / fallen-back counts (IHT_BOUNDED_STATS)."""
    runs = []
    monkeypatch.setenv("IHT_BOUND", bound)
    monkeypatch.setenv("IHT_BOUNDED_STATS", "1")
    for on in ("0", "1"):
        monkeypatch.setenv("IHT_BOUNDED", on)
        sol = iht.Solver(pool, p.s, n_iter, p.mu, p.b_y, p.seed, trace=True, nrhs=B)
        sol.run(_to_dev(Y))
        torch.cuda.synchronize()
        runs.append(tuple(t.clone() for t in sol.trace_arrays()))
        sol.close()
    import re
    m = re.search(r"bounded select: decided (\d+), fell back (\d+)", capfd.readouterr().err)
    assert m, "the bounded select did not run"
    return runs, int(m.group(1)), int(m.group(2))


@pytest.mark.parametrize("B,bound", [(16, "0.5"), (64, "0.9"), (5, "0.3")])
def test_batched_bounded_select_bit_identical(B, bound, monkeypatch, capfd):
    """Bounded select (epilogue candidates + thr_bounded_select; a snapshot the list cannot
    decide is selected over all of a by the same CTA) against the cluster kernel alone: every
    iterate of every snapshot bit-identical (both are exact H_s of the same fp32 a), and the
    bounded path decides most snapshot-iterations after the first."""
    n_iter = 24
    p, Y = _radio_batch(B, n_iter=n_iter, K=40)
    pool = iht.quantize(_to_dev(p.phi), p.b_phi, 0, p.seed, list(range(p.K)), float(OQ.scale_c(p.phi)))
    (off, on), dec, fb = _bounded_runs(pool, p, Y, B, n_iter, monkeypatch, capfd, bound)
    for a, b in zip(off, on):
        assert torch.equal(a, b)
    assert dec + fb == B * n_iter
    assert fb >= B                          # iteration 1 (x = 0) always falls back
    assert dec >= B * n_iter // 2, (dec, fb)


def test_batched_bounded_select_nan_snapshot(monkeypatch, capfd):
    """A NaN snapshot falls back (its candidates overflow / carry NaN) and reports nnz = -1;
    the others are unaffected and identical to the cluster-only run."""
    B, n_iter = 8, 6
    p, Y = _radio_batch(B, n_iter=n_iter, K=12)
    Y = Y.copy()
    Y[3, 5] = np.nan
    pool = iht.quantize(_to_dev(p.phi), p.b_phi, 0, p.seed, list(range(p.K)), float(OQ.scale_c(p.phi)))
    (off, on), dec, fb = _bounded_runs(pool, p, Y, B, n_iter, monkeypatch, capfd)
    for a, b in zip(off, on):
        assert torch.equal(a, b)
    assert int(on[2][n_iter - 1, 3]) == -1


def test_config5_bounded_select_bit_identical(monkeypatch, capfd):
    """The same at BASELINE config 5's full shape (64 snapshots of the 2304 x 65536 radio Phi,
    2-bit, K = 2 copies), 40 iterations."""
    from paper_1802_04907_b200.problem import build_pool
    p5 = G.config_problem(5, K=2)
    B, n_iter = 64, 40
    Y = np.ascontiguousarray(p5.meta["batch_y"][:, :B].T)
    pool, _, _, _, _ = build_pool(p5, 0, 1, _dev(), False, shard="cols")
    (off, on), dec, fb = _bounded_runs(pool, p5, Y, B, n_iter, monkeypatch, capfd)
    for a, b in zip(off, on):
        assert torch.equal(a, b)
    print(f"config 5 bounded select: decided {dec}, fell back {fb} of {B * n_iter}")
    assert dec >= B * n_iter // 2, (dec, fb)
