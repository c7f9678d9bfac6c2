"""GPU parity: the CUDA path (through the C ABI) against the float64 CPU oracle.

Bar (north star / SURVEY 8(c)): codes bit-exact; r, g, x within 1e-4 relative l2
per iteration; supports identical whenever the oracle's margin at the s-th
position exceeds 1e-5 |a|_(s) (otherwise logged as a near-tie).  Shapes span
several tiles with ragged tails; edge cases cover empty/degenerate inputs.
"""
import ctypes
import re

import numpy as np
import pytest
import torch

from oracle import iht as OI
from oracle import quantize as OQ
from paper_1802_04907_b200 import iht
from workloads import gen as G

from helpers import check_trajectory, rel_l2, stack, unpack_strips, pad_rows_of_strips, unstack

pytestmark = pytest.mark.gpu
TOL = 1e-4
MIN_CHECKED = 10      # free-running comparisons may never be vacuous
SEED = 0x1802_0490_7ABC


def dev():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch.device("cuda:0")


def _phi(M, N, cplx, seed=0):
    rng = np.random.default_rng(seed)
    if cplx:
        return (rng.standard_normal((M, N)) + 1j * rng.standard_normal((M, N))).astype(np.complex64)
    return rng.standard_normal((M, N)).astype(np.float32)


def _to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev())


# ------------------------------------------------------------------------- (a1) (a2) (a3)
@pytest.mark.parametrize("M,N,cplx,bits,mode", [
    (256, 1024, False, 4, 0),      # config 1 shape
    (300, 1001, False, 2, 0),      # ragged rows and columns
    (300, 1001, False, 8, 0),
    (100, 1024, True, 2, 0),       # complex (radio-like), two planes
    (257, 64, False, 4, 1),        # odd level mode
    (513, 37, True, 8, 0),
    (1, 5, False, 2, 0),           # degenerate
])
def test_quantize_codes_bit_exact(M, N, cplx, bits, mode):
    phi = _phi(M, N, cplx, seed=M + N)
    c = OQ.scale_c(phi)
    c_dev = iht.absmax(_to_dev(phi))
    assert np.float32(c_dev.item()) == c                       # (a1) exact
    copy_ids = [0, 1, 7, 399]
    copies = iht.quantize(_to_dev(phi), bits, mode, SEED, copy_ids, float(c))
    torch.cuda.synchronize()
    planes = 2 if cplx else 1
    for cid, cp in zip(copy_ids, copies):
        got = unpack_strips(cp.codes.cpu().numpy(), M, N, planes, bits)
        ref, _ = OQ.quantize_matrix(phi, bits, mode, SEED, cid, c=c)
        np.testing.assert_array_equal(got, ref)
        assert not pad_rows_of_strips(cp.codes.cpu().numpy(), M, N, planes, bits).any()


def test_quantize_rows_blockwise_equals_whole():
    M, N = 1000, 300
    phi = _phi(M, N, False, seed=3)
    c = float(OQ.scale_c(phi))
    whole = iht.quantize(_to_dev(phi), 4, 0, SEED, [5, 6], c)
    blk = [iht.new_copy(M, N, 1, 4, 0, SEED, cid, c, device=dev()) for cid in (5, 6)]
    for r0 in (0, 256, 512, 768):
        r1 = min(M, r0 + 256)
        iht.quantize_rows(_to_dev(phi[r0:r1]), blk, r0)
    torch.cuda.synchronize()
    for a, b in zip(whole, blk):          # compare the real columns (pad-column bytes are unspecified)
        np.testing.assert_array_equal(unpack_strips(a.codes.cpu().numpy(), M, N, 1, 4),
                                      unpack_strips(b.codes.cpu().numpy(), M, N, 1, 4))


def test_absmax_nan():
    t = torch.ones(1000, device=dev())
    t[517] = float("nan")
    assert np.isnan(iht.absmax(t).item())


@pytest.mark.parametrize("cplx,bits", [(False, 8), (True, 8), (False, 4)])
def test_quantize_vec_bit_exact(cplx, bits):
    M = 900 if cplx else 1000
    rng = np.random.default_rng(bits)
    y = (rng.standard_normal(M) + 1j * rng.standard_normal(M)).astype(np.complex64) if cplx else \
        rng.standard_normal(M).astype(np.float32)
    yd = _to_dev(y)
    c_dev = iht.absmax(yd)
    yhat, codes = iht.quantize_vec(yd, bits, 0, SEED, c_dev, with_codes=True)
    ref_codes, c = OQ.quantize_vector(y, bits, 0, SEED)
    assert np.float32(c_dev.item()) == c
    np.testing.assert_array_equal(codes.cpu().numpy().reshape(ref_codes.shape), ref_codes)
    ref = stack(OQ.dequantize(ref_codes, c, bits, 0), M)
    assert rel_l2(yhat.cpu().numpy(), ref) < 1e-6


# ------------------------------------------------------------------------- (a4) forward
@pytest.mark.parametrize("M,N,cplx,bits,s", [(256, 1024, False, 4, 16), (300, 1001, False, 2, 37),
                                              (100, 1024, True, 2, 9), (513, 200, False, 8, 200),
                                              (4096, 2048, False, 4, 128)])
def test_forward_parity(M, N, cplx, bits, s):
    phi = _phi(M, N, cplx, seed=1)
    c = OQ.scale_c(phi)
    (F,) = iht.quantize(_to_dev(phi), bits, 0, SEED, [3], float(c))
    Fd = OQ.dequantize(OQ.quantize_matrix(phi, bits, 0, SEED, 3, c=c)[0], c, bits, 0)
    rng = np.random.default_rng(s)
    x_idx = np.sort(rng.choice(N, s, replace=False))
    x_val = rng.standard_normal(s).astype(np.float32)
    yh = (rng.standard_normal(M) + (1j * rng.standard_normal(M) if cplx else 0)).astype(np.complex128 if cplx else np.float64)
    yh32 = stack(yh, M).astype(np.float32)
    r = iht.forward(F, _to_dev(x_idx.astype(np.int32)), _to_dev(x_val), _to_dev(np.array([s], np.int32)),
                    _to_dev(yh32))
    ref = OI.forward(Fd, x_idx, x_val.astype(np.float64), unstack(yh32, M, 2 if cplx else 1))
    got = r.cpu().numpy()
    assert rel_l2(unstack(got, M, 2 if cplx else 1), ref) < TOL
    assert not np.any(got[stack(np.ones(M) * (1 + 1j if cplx else 1), M) == 0])   # pads stay 0
    # empty support: r = y-hat
    r0 = iht.forward(F, _to_dev(x_idx.astype(np.int32)), _to_dev(x_val), _to_dev(np.array([0], np.int32)),
                     _to_dev(yh32))
    np.testing.assert_array_equal(r0.cpu().numpy(), yh32)


@pytest.mark.parametrize("M,N,cplx,bits,s,nnz", [(40000, 600, False, 4, 600, 600), (40000, 600, False, 4, 300, 300),
                                                  (40000, 600, False, 4, 600, 555), (80000, 400, False, 2, 400, 400),
                                                  (20000, 1100, False, 8, 1100, 1037), (20000, 300, True, 4, 300, 300)])
def test_forward_split_parity(M, N, cplx, bits, s, nnz, monkeypatch):
    """The row-block x column-group forward (IHT_FWD_SPLIT=1; measured slower than forward_kernel
    at config 4, so not the default) on >= 296 row blocks (config-4-like rows) incl. G > 1
    column groups summed by the last CTA of each row block, a ragged nnz < max_nnz, 2/4/8 bits
    and complex rows: r within 1e-4 of the oracle's forward; repeated calls reuse the zeroed
    workspace (the arrival counters are reset by the kernel) and give identical bits."""
    monkeypatch.setenv("IHT_FWD_SPLIT", "1")
    phi = _phi(M, N, cplx, seed=5)
    c = OQ.scale_c(phi)
    (F,) = iht.quantize(_to_dev(phi), bits, 0, SEED, [1], float(c))
    assert iht.load().iht_forward_ws_bytes(ctypes.byref(F.desc), s) >= (0 if s <= 300 else 1)
    Fd = OQ.dequantize(OQ.quantize_matrix(phi, bits, 0, SEED, 1, c=c)[0], c, bits, 0)
    del phi
    rng = np.random.default_rng(s + nnz)
    x_idx = np.sort(rng.choice(N, s, replace=False))
    x_val = rng.standard_normal(s).astype(np.float32)
    yh = (rng.standard_normal(M) + (1j * rng.standard_normal(M) if cplx else 0)).astype(np.complex128 if cplx else np.float64)
    yh32 = stack(yh, M).astype(np.float32)
    args = (_to_dev(x_idx.astype(np.int32)), _to_dev(x_val), _to_dev(np.array([nnz], np.int32)), _to_dev(yh32))
    lib = iht.load()
    ws_bytes = lib.iht_forward_ws_bytes(ctypes.byref(F.desc), s)
    ws = torch.zeros(max(ws_bytes, 1), dtype=torch.uint8, device=dev())
    outs = []
    for _ in range(2):                           # the same workspace twice: counters back at zero
        r = torch.empty_like(args[3])
        assert lib.iht_forward(ctypes.byref(F.desc), iht._ptr(args[0]), iht._ptr(args[1]), iht._ptr(args[2]), s,
                               iht._ptr(args[3]), iht._ptr(r), iht._ptr(ws), ws_bytes, None) == 0
        torch.cuda.synchronize()
        outs.append(r.cpu().numpy())
    np.testing.assert_array_equal(outs[0], outs[1])
    if ws_bytes:                                 # the arrival counters (tail of the workspace) are back at 0
        nrb = F.desc.strip_bytes // 4 // 16
        assert int(ws[ws_bytes - 4 * nrb:ws_bytes].count_nonzero().item()) == 0
    ref = OI.forward(Fd, x_idx[:nnz], x_val[:nnz].astype(np.float64), unstack(yh32, M, 2 if cplx else 1))
    assert rel_l2(unstack(outs[0], M, 2 if cplx else 1), ref) < TOL
    assert not np.any(outs[0][stack(np.ones(M) * (1 + 1j if cplx else 1), M) == 0])   # pads stay 0


# ------------------------------------------------------------------------- (a5) adjoint
ADJ_CASES = [(256, 1024, False, 4), (300, 1001, False, 2), (300, 1001, False, 8), (100, 1024, True, 2),
             (2304, 3000, True, 2), (4500, 777, False, 4), (9000, 260, False, 8), (70000, 40, False, 4)]


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("M,N,cplx,bits", ADJ_CASES)
def test_adjoint_parity(M, N, cplx, bits, variant):
    phi = _phi(M, N, cplx, seed=2)
    c = OQ.scale_c(phi)
    (A,) = iht.quantize(_to_dev(phi), bits, 0, SEED, [11], float(c))
    Ad = OQ.dequantize(OQ.quantize_matrix(phi, bits, 0, SEED, 11, c=c)[0], c, bits, 0)
    rng = np.random.default_rng(M)
    r = rng.standard_normal(M) + (1j * rng.standard_normal(M) if cplx else 0)
    r[: M // 7] *= 1e-3                 # dynamic range inside fixed-point chunks
    r32 = stack(r, M).astype(np.float32)
    g = iht.adjoint(A, _to_dev(r32), variant=variant).cpu().numpy()
    ref = OI.adjoint(Ad, unstack(r32, M, 2 if cplx else 1))
    assert rel_l2(g, ref) < TOL, rel_l2(g, ref)


def test_adjoint_zero_and_tiny_r():
    M, N = 512, 300
    phi = _phi(M, N, False, seed=4)
    c = OQ.scale_c(phi)
    (A,) = iht.quantize(_to_dev(phi), 4, 0, SEED, [0], float(c))
    z = torch.zeros(iht.vec_len(M, 1), device=dev())
    assert torch.count_nonzero(iht.adjoint(A, z, 0)) == 0
    Ad = OQ.dequantize(OQ.quantize_matrix(phi, 4, 0, SEED, 0, c=c)[0], c, 4, 0)
    for scale in (1e-30, 1e20):
        r = (np.random.default_rng(1).standard_normal(M) * scale).astype(np.float32)
        g = iht.adjoint(A, _to_dev(stack(r, M).astype(np.float32)), 0).cpu().numpy()
        assert rel_l2(g, OI.adjoint(Ad, r.astype(np.float64))) < TOL


# ------------------------------------------------------------------------- (a6) threshold
def _thr(x_idx, x_val, g, mu, s):
    xi = _to_dev(np.asarray(x_idx, np.int32)) if len(x_idx) else torch.zeros(max(s, 1), dtype=torch.int32, device=dev())
    xv = _to_dev(np.asarray(x_val, np.float32)) if len(x_val) else torch.zeros(max(s, 1), device=dev())
    nnz = _to_dev(np.array([len(x_idx)], np.int32))
    oi, ov, on = iht.threshold(xi, xv, nnz, _to_dev(np.asarray(g, np.float32)), mu, s)
    n = int(on.item())
    if n < 0:
        return None, None
    return oi[:n].cpu().numpy(), ov[:n].cpu().numpy()


def _a32(x_idx, x_val, g, mu):
    a = (np.float32(mu) * np.asarray(g, np.float32)).astype(np.float32)
    a[np.asarray(x_idx, np.int64)] = (np.asarray(x_val, np.float32) + a[np.asarray(x_idx, np.int64)]).astype(np.float32)
    return a


@pytest.mark.parametrize("N,s", [(1024, 16), (16384, 128), (262144, 1024), (1001, 37), (5, 3), (1, 1),
                                 (100, 100), (100, 150), (3000, 0), (131073, 64), (262145, 1024),   # fused cluster
                                 (262144, 5000), (20000, 4500),        # fused, > 4096 candidates: per-pass path
                                 (300000, 100), (300000, 7000),                                    # grid path
                                 (131072, 1024), (200000, 3000), (262144, 1)])                     # grid path
def test_threshold_exact_selection(N, s):
    """Selection on identical fp32 a is exact: GPU H_s = oracle H_s of the same a."""
    rng = np.random.default_rng(N + s)
    g = rng.standard_normal(N).astype(np.float32)
    k = min(s, N)
    x_idx = np.sort(rng.choice(N, k, replace=False)) if k else np.zeros(0, np.int64)
    x_val = rng.standard_normal(k).astype(np.float32)
    idx, val = _thr(x_idx, x_val, g, 0.7, s)
    a = _a32(x_idx, x_val, g, 0.7)
    ri, rv = OI.hard_threshold(a.astype(np.float64), s)
    np.testing.assert_array_equal(idx, ri)
    np.testing.assert_array_equal(val, rv.astype(np.float32))


def test_threshold_ties_and_zeros():
    g = np.zeros(4096, np.float32)
    g[[5, 9, 100, 2000, 4095]] = [2.0, -2.0, 2.0, 1.0, -2.0]         # ties at |2|
    idx, val = _thr([], [], g, 1.0, 3)
    assert idx.tolist() == [5, 9, 100]                               # lowest indices win
    idx, val = _thr([], [], g, 1.0, 10)                              # fewer nonzeros than s
    assert idx.tolist() == [5, 9, 100, 2000, 4095]
    idx, val = _thr([], [], np.zeros(100, np.float32), 1.0, 5)       # all zero -> empty
    assert idx.size == 0
    many = np.full(70000, 0.5, np.float32)                           # massive tie
    idx, _ = _thr([], [], many, 1.0, 1000)
    assert idx.tolist() == list(range(1000))
    many = np.full(262144, 0.5, np.float32)                          # massive tie on the grid path
    idx, _ = _thr([], [], many, 1.0, 1000)
    assert idx.tolist() == list(range(1000))
    crowd = np.full(262144, 0.01, np.float32)                        # a crowded bin just below the top
    crowd[::3] = 0.75
    crowd[::3000] = 1.0
    idx, _ = _thr([], [], crowd, 1.0, 500)
    ri, _ = OI.hard_threshold(crowd.astype(np.float64), 500)
    assert idx.tolist() == ri.tolist()


def _iterate_like(N, s, rng, jump=1.0, crowd=0):
    """H_s input shaped like a solver iteration: x = H_s(a0) (so min |x| is the previous
    threshold), then a new g; `jump` scales g (the threshold moves far), `crowd` places that
    many keys just below the previous threshold (more candidates than the gather holds)."""
    a0 = rng.standard_normal(N).astype(np.float32)
    xi, xv = OI.hard_threshold(a0.astype(np.float64), s)
    xv = xv.astype(np.float32)
    g = (0.3 * jump * rng.standard_normal(N)).astype(np.float32)
    if crowd:
        thr = np.float32(np.min(np.abs(xv)))
        pos = rng.choice(np.setdiff1d(np.arange(N), xi), crowd, replace=False)
        g[pos] = np.float32(0.95) * thr * np.where(rng.random(crowd) < 0.5, 1, -1).astype(np.float32)
    return xi, xv, g


@pytest.mark.parametrize("N,s,jump,crowd", [(131072, 1024, 1.0, 0), (262144, 1024, 1.0, 0), (262144, 1024, 30.0, 0),
                                            (262144, 1024, 1.0, 12000), (300000, 7000, 1.0, 0),
                                            (262145, 4000, 0.1, 0), (262144, 64, 1.0, 0)])
def test_threshold_onepass_iteration_shaped(N, s, jump, crowd):
    """The one-launch grid select (thr_onepass: histogram, grid barrier, candidates, last-CTA
    finish) on iteration-shaped inputs, incl. a threshold jump and a crowded bin that
    overflows the gather: exact H_s of the same fp32 a."""
    rng = np.random.default_rng(N + s + int(jump) + crowd)
    xi, xv, g = _iterate_like(N, s, rng, jump, crowd)
    idx, val = _thr(xi, xv, g, 1.0, s)
    a = _a32(xi, xv, g, 1.0)
    ri, rv = OI.hard_threshold(a.astype(np.float64), s)
    np.testing.assert_array_equal(idx, ri)
    np.testing.assert_array_equal(val, rv.astype(np.float32))


def test_threshold_onepass_ties_at_threshold():
    """Ties at the selected key spread over many tiles of the grid select: the lowest
    indices win across tile boundaries (reading c15)."""
    N, s = 262144, 1000
    rng = np.random.default_rng(7)
    xi = np.sort(rng.choice(N, s, replace=False))
    xv = np.full(s, 1.0, np.float32)
    g = np.zeros(N, np.float32)
    g[xi] = 0.0
    tie = np.sort(rng.choice(np.setdiff1d(np.arange(N), xi), 3000, replace=False))
    g[tie] = 0.95                                    # 3000 keys at 0.95 compete for nothing; x stays
    xv[:200] = 0.5                                   # 200 of x fall below the ties: 200 ties at 0.95 are taken
    idx, val = _thr(xi, xv, g, 1.0, s)
    a = _a32(xi, xv, g, 1.0)
    ri, rv = OI.hard_threshold(a.astype(np.float64), s)
    np.testing.assert_array_equal(idx, ri)
    np.testing.assert_array_equal(val, rv.astype(np.float32))


@pytest.mark.parametrize("N", [16384, 65536, 262144])
def test_threshold_ties_across_cluster(N):
    """Gathered select (few candidates): ties at T spread over every CTA of the cluster;
    the lowest indices win across CTA boundaries."""
    rng = np.random.default_rng(N)
    g = (0.01 * rng.standard_normal(N)).astype(np.float32)
    tie = np.sort(rng.choice(N, 300, replace=False))
    g[tie] = np.where(rng.random(300) < 0.5, 2.0, -2.0).astype(np.float32)
    big = tie[::7][:20]
    g[big] = 3.0
    idx, val = _thr([], [], g, 1.0, 100)
    ri, rv = OI.hard_threshold(g.astype(np.float64), 100)
    np.testing.assert_array_equal(idx, ri)
    rest = [i for i in tie if i not in set(big.tolist())][:80]
    assert sorted(big.tolist() + rest) == idx.tolist()


@pytest.mark.parametrize("N", [1000, 262144])
def test_threshold_nan_domain_error(N):
    g = np.ones(N, np.float32)
    g[10] = np.nan
    idx, _ = _thr([], [], g, 1.0, 4)
    assert idx is None


# ------------------------------------------------------------------------- solver
def _pool(phi, bits, K, c, seed, mode=0):
    return iht.quantize(_to_dev(phi), bits, mode, seed, list(range(K)), float(c))


def _support_ok(rec, got_idx, s):
    a = np.abs(rec.a)
    ks = np.sort(a)[::-1]
    kth = ks[min(s, a.size) - 1] if s > 0 else 0.0
    if rec.margin > 1e-5 * max(kth, 1e-30):
        return list(got_idx) == list(rec.x_idx), True
    return True, False


CASES = {
    "config1": lambda: G.config_problem(1, K=200),
    "gauss2bit": lambda: G.gaussian_problem(1024, 4096, 40, cfg_id=21, values="sign", b_phi=2, n_iter=30,
                                            mu=0.15, K=60),
    "radio": lambda: G.radio_problem(cfg_id=23, A=12, grid=48, n_src=10, n_iter=30, K=60),
    "gauss8bit": lambda: G.gaussian_problem(700, 3001, 20, cfg_id=22, b_phi=8, n_iter=25, K=4),
    # 3 K-ranges of the int8-MMA adjoint: the solver sums the split-K partials inside the
    # fused threshold (no reduce kernel)
    "splitk": lambda: G.gaussian_problem(2100, 4096, 20, cfg_id=24, b_phi=4, n_iter=15, mu=0.6, K=30),
    # N >= 131072: H_s on the grid path (T1 - T3 over every SM) inside the solver graph
    "gridsel": lambda: G.gaussian_problem(512, 140000, 24, cfg_id=25, b_phi=4, n_iter=10, mu=0.5, K=20),
}


@pytest.mark.parametrize("case", list(CASES))
def test_teacher_forced_iterations(case):
    """Feed the oracle's x^[n] into the GPU forward / adjoint / threshold each iteration."""
    p = CASES[case]()
    n_iter = min(p.n_iter, 40)
    ref = OI.qniht(p.phi, p.y, p.s, n_iter, p.mu, p.b_phi, p.b_y, p.seed, p.K)
    c = OQ.scale_c(p.phi)
    pool = _pool(p.phi, p.b_phi, min(p.K, 2 * n_iter), c, p.seed)
    planes = 2 if p.complex else 1
    yd = _to_dev(p.y)
    c_y = iht.absmax(yd)
    yhat, _ = iht.quantize_vec(yd, p.b_y, 0, p.seed, c_y)
    assert rel_l2(yhat.cpu().numpy(), stack(ref.y_hat, p.M)) < 1e-6
    x_idx, x_val = np.zeros(0, np.int64), np.zeros(0)
    checked = 0
    for rec in ref.trace:
        xi = _to_dev(np.resize(x_idx.astype(np.int32), max(p.s, 1)))
        xv = _to_dev(np.resize(x_val.astype(np.float32), max(p.s, 1)))
        nz = _to_dev(np.array([len(x_idx)], np.int32))
        r = iht.forward(pool[rec.fwd_copy], xi, xv, nz, yhat)
        assert rel_l2(unstack(r.cpu().numpy(), p.M, planes), rec.r, floor=1e-6 * np.linalg.norm(ref.y_hat)) < TOL
        r_or = _to_dev(stack(rec.r, p.M).astype(np.float32))
        g = iht.adjoint(pool[rec.adj_copy], r_or)
        assert rel_l2(g.cpu().numpy(), rec.g) < TOL
        oi, ov, on = iht.threshold(xi, xv, nz, _to_dev(rec.g.astype(np.float32)), p.mu, p.s)
        n = int(on.item())
        gi, gv = oi[:n].cpu().numpy(), ov[:n].cpu().numpy()
        ok, strict = _support_ok(rec, gi, p.s)
        assert ok, f"iteration {rec.n}: support differs with margin {rec.margin}"
        if strict:
            checked += 1
            assert rel_l2(gv, rec.x_val, floor=1e-30) < TOL
        x_idx, x_val = rec.x_idx, rec.x_val
    assert checked >= len(ref.trace) // 2


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("graph,fused", [(True, True), (True, False), (False, False)])
def test_free_running_solver(case, graph, fused):
    """Whole solve through iht_solver (CUDA graph) vs the oracle trajectory: identical
    supports and x within 1e-4 up to the first near-tie; final support identical
    when no near-tie occurred."""
    p = CASES[case]()
    n_iter = min(p.n_iter, 40)
    ref = OI.qniht(p.phi, p.y, p.s, n_iter, p.mu, p.b_phi, p.b_y, p.seed, p.K)
    c = OQ.scale_c(p.phi)
    pool = _pool(p.phi, p.b_phi, min(p.K, 2 * n_iter), c, p.seed)
    sol = iht.Solver(pool, p.s, n_iter, p.mu, p.b_y, p.seed, trace=True, use_graph=graph,
                     fused="force" if fused else False)
    assert sol.fused == fused                 # every case fits the fused persistent kernel
    sol.run(_to_dev(p.y))
    idx, val, nnz = sol.trace_arrays()
    checked = check_trajectory(ref.trace, idx, val, nnz, p.s, TOL)
    # no escape: every iteration up to the oracle's first near-tie meets the bar, and the
    # comparison is never vacuous (the cases are chosen so that no near-tie comes early)
    assert checked >= min(len(ref.trace), MIN_CHECKED), f"only {checked} iterations before a near-tie"
    if checked == len(ref.trace):          # no near-tie at all: the final support is identical
        fi, fv, fn = sol.run(_to_dev(p.y))
        torch.cuda.synchronize()
        k = int(fn.item())
        assert fi[:k].cpu().numpy().tolist() == ref.x_idx.tolist()
        assert rel_l2(fv[:k].cpu().numpy(), ref.x_val, floor=1e-30) < TOL
    sol.close()


@pytest.mark.parametrize("case", ["config1", "gauss2bit", "radio", "gauss8bit", "splitk"])
def test_fused_bounded_candidates_bit_identical(case, capfd, monkeypatch):
    """The fused solver's bounded-candidate select (candidates = keys >= 0.7 x the previous
    threshold, written before barrier 2; when at least s of them exist, the histogram, S1 and
    barrier 3 are skipped and S2 selects from them alone) is exact: every iterate is
    bit-identical to the unbounded path (IHT_FUSED_NOBOUND=1), and the bounded path is actually
    taken (phase timeline: barrier 3 skipped)."""
    p = CASES[case]()
    n_iter = min(p.n_iter, 40)
    c = OQ.scale_c(p.phi)
    pool = _pool(p.phi, p.b_phi, min(p.K, 2 * n_iter), c, p.seed)
    y = _to_dev(p.y)
    runs = []
    for env in ({"IHT_FUSED_NOBOUND": "1"}, {"IHT_FUSED_TL": "0"}):
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        sol = iht.Solver(pool, p.s, n_iter, p.mu, p.b_y, p.seed, trace=True, fused="force")
        assert sol.fused
        sol.run(y)
        torch.cuda.synchronize()
        runs.append(tuple(t.clone() for t in sol.trace_arrays()))
        sol.close()
        for k in env:
            monkeypatch.delenv(k)
    for a, b in zip(runs[0], runs[1]):
        assert torch.equal(a, b)
    err = capfd.readouterr().err
    m = re.search(r"B3 skipped (\d+)/(\d+)", err)
    assert m, err[-2000:]
    assert int(m.group(1)) >= 1, f"bounded path never taken: {m.group(0)}"


def test_solver_host_io_and_determinism():
    p = CASES["gauss8bit"]()
    c = OQ.scale_c(p.phi)
    pool = _pool(p.phi, p.b_phi, p.K, c, p.seed)
    sol = iht.Solver(pool, p.s, p.n_iter, p.mu, p.b_y, p.seed)
    yh = torch.from_numpy(p.y).pin_memory()
    oi = torch.empty(p.s, dtype=torch.int32).pin_memory()
    ov = torch.empty(p.s, dtype=torch.float32).pin_memory()
    on = torch.empty(1, dtype=torch.int32).pin_memory()
    sol.run_host(yh, oi, ov, on)
    a = (oi.clone(), ov.clone(), int(on))
    sol.run_host(yh, oi, ov, on)
    assert torch.equal(a[0], oi) and torch.equal(a[1], ov) and a[2] == int(on)     # bit-reproducible
    di, dv, dn = sol.run(_to_dev(p.y))
    torch.cuda.synchronize()
    assert torch.equal(di.cpu(), oi) and torch.equal(dv.cpu(), ov)
    sol.close()


def test_solver_world1_row_shard_path():
    """The row-sharded code path (c_y max-all-reduce, g sum-all-reduce through NCCL, and the
    host-driven shrink loop of the adaptive step) at world size 1 gives bit-identical results
    to the plain run."""
    p = CASES["gauss8bit"]()
    c = OQ.scale_c(p.phi)
    pool = _pool(p.phi, p.b_phi, p.K, c, p.seed)
    comm = iht.Comm(0, 1, 0)
    try:
        for adaptive in (False, True):
            ref = iht.Solver(pool, p.s, 12, p.mu, p.b_y, p.seed, adaptive=adaptive, fused=False)
            ri, rv, rn = [t.cpu().clone() for t in ref.run(_to_dev(p.y))]
            sol = iht.Solver(pool, p.s, 12, p.mu, p.b_y, p.seed, comm=comm, adaptive=adaptive)
            gi, gv, gn = sol.run(_to_dev(p.y))
            torch.cuda.synchronize()
            assert torch.equal(gi.cpu(), ri) and torch.equal(gv.cpu(), rv) and torch.equal(gn.cpu(), rn)
            sol.close()
            ref.close()
    finally:
        comm.close()


def test_solver_edge_cases():
    """n* = 0 returns x = 0 (empty support); s = 0 keeps nothing; a NaN in y reaches
    H_s and is reported as IHT_EDOMAIN by the host-IO run."""
    p = CASES["gauss8bit"]()
    c = OQ.scale_c(p.phi)
    pool = _pool(p.phi, p.b_phi, 2, c, p.seed)
    sol = iht.Solver(pool, p.s, 0, p.mu, p.b_y, p.seed)
    _, _, n = sol.run(_to_dev(p.y))
    torch.cuda.synchronize()
    assert int(n.item()) == 0
    sol.close()
    sol = iht.Solver(pool, 0, 5, p.mu, p.b_y, p.seed)
    _, _, n = sol.run(_to_dev(p.y))
    torch.cuda.synchronize()
    assert int(n.item()) == 0
    sol.close()
    y = p.y.copy()
    y[3] = np.nan
    sol = iht.Solver(pool, p.s, 3, p.mu, p.b_y, p.seed)
    oi = torch.empty(p.s, dtype=torch.int32).pin_memory()
    ov = torch.empty(p.s, dtype=torch.float32).pin_memory()
    on = torch.empty(1, dtype=torch.int32).pin_memory()
    with pytest.raises(iht._lib.IhtError) as e:
        sol.run_host(torch.from_numpy(y).pin_memory(), oi, ov, on)
    assert e.value.status == iht._lib.IHT_EDOMAIN
    sol.close()
