"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times
(paper_1802_04907_b200.problem.build_pool + the same kernels/plans), on outputs the
oracle can compute one by one.

* config 2 (4096 x 16384, 2-bit, K = 400 copies): codes of whole copies bit-exact; two
  teacher-forced iterations (forward, adjoint, threshold) against the dense oracle.
* config 5 (2304 x 65536 complex radio, 2-bit, B = 64, K = 400): sampled code blocks bit-exact,
  the batched tcgen05 adjoint on sampled pixels, the batched forward on true supports, the
  exact top-64 of all 64 snapshots; config 3 (its snapshot 0) through the GEMV adjoint.
* config 4 (65536 x 262144, 4-bit, K = 2, 16 GiB of codes): the device absmax equals
  the oracle's c (tests/golden/config4_scale.json, written by scripts/golden_config4.py
  from oracle/ only); random code tiles bit-exact; adjoint on 64 sampled columns,
  forward on 64 sampled rows against the oracle computed column/row-wise; the full
  top-1024 selection over N = 262144 exact against oracle H_s of the same fp32 a.
"""
import json
import os

import numpy as np
import pytest
import torch

from oracle import iht as OI
from oracle import quantize as OQ
from paper_1802_04907_b200 import iht
from paper_1802_04907_b200.problem import build_pool
from workloads import gen as G

from helpers import rel_l2, stack, unpack_strips, unstack

pytestmark = pytest.mark.gpu
TOL = 1e-4
GOLDEN4 = os.path.join(os.path.dirname(__file__), "golden", "config4_scale.json")


def _dev():
    return torch.device("cuda:0")


def _to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(_dev())


def _tile_codes(cp, rows, cols, planes, bits, r0, nr, c0, nc):
    """codes (planes, nr, nc) of rows [r0, r0+nr) x cols [c0, c0+nc) from a device copy
    (reads only the needed 16-column tiles)."""
    sb = iht.strip_bytes(rows, planes, bits)
    t0, t1 = c0 // 16, (c0 + nc + 15) // 16
    raw = cp.codes[t0 * 16 * sb:t1 * 16 * sb].cpu().numpy()
    full = unpack_strips(raw, rows, (t1 - t0) * 16, planes, bits)
    return full[:, r0:r0 + nr, c0 - t0 * 16:c0 - t0 * 16 + nc]


@pytest.fixture(scope="module")
def config2():
    p = G.config_problem(2)                     # K = 2 n* = 400
    pool, c, _, rows, row0 = build_pool(p, 0, 1, _dev(), False)
    torch.cuda.synchronize()
    return p, pool, c


def test_config2_codes_and_teacher_forced(config2):
    p, pool, c = config2
    assert len(pool) == 400
    c_ref = OQ.scale_c(p.phi)
    assert np.float32(c) == c_ref
    copies = {}
    for cid in (0, 1, 2, 3):           # iterations 1, 2 use copies 0..3 (adjoint 2n-2, forward 2n-1)
        ref, _ = OQ.quantize_matrix(p.phi, p.b_phi, 0, p.seed, cid, c=c_ref)
        got = _tile_codes(pool[cid], p.M, p.N, 1, p.b_phi, 0, p.M, 0, p.N)
        np.testing.assert_array_equal(got, ref)
        copies[cid] = OQ.dequantize(ref, c_ref, p.b_phi, 0)
    # last copy of the pool on a sample of columns
    ref, _ = OQ.quantize_matrix(p.phi[:, 8000:8100], p.b_phi, 0, p.seed, 399, c=c_ref, col_offset=8000)
    np.testing.assert_array_equal(_tile_codes(pool[399], p.M, p.N, 1, p.b_phi, 0, p.M, 8000, 100), ref)
    # two teacher-forced iterations at full size
    yd = _to_dev(p.y)
    yhat, _ = iht.quantize_vec(yd, p.b_y, 0, p.seed, iht.absmax(yd))
    y_codes, c_y = OQ.quantize_vector(p.y, p.b_y, 0, p.seed)
    y_hat = OQ.dequantize(y_codes, c_y, p.b_y, 0)
    x_idx, x_val = np.zeros(0, np.int64), np.zeros(0)
    for n in (1, 2):
        a_id, f_id = 2 * n - 2, 2 * n - 1
        r_ref = OI.forward(copies[f_id], x_idx, x_val, y_hat)
        xi = _to_dev(np.resize(x_idx.astype(np.int32), p.s))
        xv = _to_dev(np.resize(x_val.astype(np.float32), p.s))
        nz = _to_dev(np.array([len(x_idx)], np.int32))
        r = iht.forward(pool[f_id], xi, xv, nz, yhat)
        assert rel_l2(unstack(r.cpu().numpy(), p.M, 1), r_ref) < TOL
        g_ref = OI.adjoint(copies[a_id], r_ref)
        g = iht.adjoint(pool[a_id], _to_dev(stack(r_ref, p.M).astype(np.float32)))
        assert rel_l2(g.cpu().numpy(), g_ref) < TOL
        a = np.zeros(p.N)
        a[x_idx] = x_val
        a = a + p.mu * g_ref
        ri, rv = OI.hard_threshold(a, p.s)
        oi, ov, on = iht.threshold(xi, xv, nz, _to_dev(g_ref.astype(np.float32)), p.mu, p.s)
        k = int(on.item())
        margin = OI.margin_at_s(a, p.s)
        if margin > 1e-5 * np.sort(np.abs(a))[::-1][p.s - 1]:
            assert oi[:k].cpu().numpy().tolist() == ri.tolist()
            assert rel_l2(ov[:k].cpu().numpy(), rv) < TOL
        x_idx, x_val = ri, rv


@pytest.fixture(scope="module")
def config4():
    if not os.path.exists(GOLDEN4):
        pytest.skip("golden scale missing (scripts/golden_config4.py)")
    gold = json.load(open(GOLDEN4))
    p = G.config_problem(4)                     # K = 2, materialize = False
    p.K = 2
    pool, c, _, rows, row0 = build_pool(p, 0, 1, _dev(), False)
    torch.cuda.synchronize()
    return p, pool, c, float.fromhex(gold["c_phi_hex"])


def test_config4_scale_and_code_tiles(config4):
    p, pool, c, c_gold = config4
    assert np.float32(c) == np.float32(c_gold)                        # (a1) exact
    rng = np.random.default_rng(44)
    for cid in (0, 1):
        for _ in range(6):
            r0 = int(rng.integers(0, p.M // 256)) * 256
            c0 = int(rng.integers(0, p.N - 64))
            phi = G.gaussian_block(p.phi_key, p.N, r0, 256, c0, 64, p.phi_sd)
            ref, _ = OQ.quantize_matrix(phi, p.b_phi, 0, p.seed, cid, c=np.float32(c_gold),
                                        row_offset=r0, col_offset=c0)
            got = _tile_codes(pool[cid], p.M, p.N, 1, p.b_phi, r0, 256, c0, 64)
            np.testing.assert_array_equal(got, ref)


def test_config4_adjoint_forward_threshold_sampled(config4):
    p, pool, c, c_gold = config4
    c_gold = np.float32(c_gold)
    rng = np.random.default_rng(45)
    # adjoint on 64 sampled columns (oracle: whole quantised columns, one by one)
    r = rng.standard_normal(p.M).astype(np.float32) * 0.1
    r[: p.M // 9] *= 1e-3
    g = iht.adjoint(pool[0], _to_dev(stack(r, p.M).astype(np.float32))).cpu().numpy()
    cols = np.sort(rng.choice(p.N, 64, replace=False))
    g_ref = np.empty(64)
    for i, n in enumerate(cols):
        col = G.gaussian_columns(p.phi_key, p.N, 0, p.M, [n], p.phi_sd)
        q, _ = OQ.quantize_matrix(col, p.b_phi, 0, p.seed, 0, c=c_gold, col_offset=int(n))
        g_ref[i] = OI.adjoint(OQ.dequantize(q, c_gold, p.b_phi, 0), r.astype(np.float64))[0]
    assert rel_l2(g[cols], g_ref) < TOL
    # forward on 64 sampled rows with a random s-sparse x
    s = p.s
    x_idx = np.sort(rng.choice(p.N, s, replace=False))
    x_val = rng.standard_normal(s).astype(np.float32)
    yh = (rng.standard_normal(p.M) * 0.1).astype(np.float32)
    rr = iht.forward(pool[1], _to_dev(x_idx.astype(np.int32)), _to_dev(x_val), _to_dev(np.array([s], np.int32)),
                     _to_dev(stack(yh, p.M).astype(np.float32))).cpu().numpy()
    rows = np.sort(rng.choice(p.M, 64, replace=False))
    r_ref = np.empty(64)
    for i, m in enumerate(rows):
        row = G.gaussian_columns(p.phi_key, p.N, int(m), 1, x_idx, p.phi_sd)     # Phi[m, x_idx]
        q = np.empty((1, 1, s), dtype=np.uint8)
        for j, n in enumerate(x_idx):
            q[:, :, j:j + 1] = OQ.quantize_matrix(row[:, j:j + 1], p.b_phi, 0, p.seed, 1, c=c_gold,
                                                  row_offset=int(m), col_offset=int(n))[0]
        F = OQ.dequantize(q, c_gold, p.b_phi, 0)
        r_ref[i] = OI.forward(F, np.arange(s), x_val.astype(np.float64), np.array([float(yh[m])]))[0]
    assert rel_l2(rr[rows], r_ref) < TOL
    # exact top-1024 selection over N = 262144 on the fp32 a the kernel sees
    mu = np.float32(p.mu)
    xi = _to_dev(x_idx.astype(np.int32))
    xv = _to_dev(x_val)
    oi, ov, on = iht.threshold(xi, xv, _to_dev(np.array([s], np.int32)), _to_dev(g), float(mu), s)
    a32 = (mu * g).astype(np.float32)
    a32[x_idx] = (x_val + a32[x_idx]).astype(np.float32)
    ri, rv = OI.hard_threshold(a32.astype(np.float64), s)
    k = int(on.item())
    assert oi[:k].cpu().numpy().tolist() == ri.tolist()
    np.testing.assert_array_equal(ov[:k].cpu().numpy(), rv.astype(np.float32))


# ------------------------------------------------------------------------------ config 3 / 5
@pytest.fixture(scope="module")
def config5():
    """Config 5 (config 3's radio Phi, 2304 x 65536 complex, 2-bit, B = 64 snapshots) built as
    bench.py builds it (column shard of the whole Phi at world size 1, K = 400 copies)."""
    p = G.config_problem(5)
    pool, c, _, rows, row0 = build_pool(p, 0, 1, _dev(), False, shard="cols")
    torch.cuda.synchronize()
    return p, pool, c


def _radio_cols(p, cid, c, cols):
    """Oracle codes -> dequantised columns `cols` of copy cid (complex, M x len(cols))."""
    blk = np.ascontiguousarray(p.phi[:, cols])
    out = np.empty((p.M, len(cols)), np.complex128)
    for j, n in enumerate(cols):            # one column at a time: global column index n
        q, _ = OQ.quantize_matrix(blk[:, j:j + 1], p.b_phi, 0, p.seed, cid, c=c, col_offset=int(n))
        out[:, j] = OQ.dequantize(q, c, p.b_phi, 0)[:, 0]
    return out


def test_config5_codes_adjoint_forward_threshold_sampled(config5):
    p, pool, c = config5
    assert len(pool) == 400
    c_ref = OQ.scale_c(p.phi)
    assert np.float32(c) == c_ref                                          # (a1) exact
    rng = np.random.default_rng(55)
    # codes: random 64-column blocks of copies 0, 1 and 399, all rows and both planes
    for cid in (0, 1, 399):
        c0 = int(rng.integers(0, p.N - 64)) // 16 * 16
        ref, _ = OQ.quantize_matrix(np.ascontiguousarray(p.phi[:, c0:c0 + 64]), p.b_phi, 0, p.seed, cid, c=c_ref,
                                    col_offset=c0)
        np.testing.assert_array_equal(_tile_codes(pool[cid], p.M, p.N, 2, p.b_phi, 0, p.M, c0, 64), ref)
    B = p.meta["batch_y"].shape[1]
    Y = np.ascontiguousarray(p.meta["batch_y"].T)                          # (B, M)
    Yd = _to_dev(Y)
    yhat, _ = iht.quantize_vec_batched(Yd, p.b_y, 0, p.seed, iht.absmax_batched(Yd))
    # iteration 1 of every snapshot, teacher-forced: r = y-hat (x = 0), g on 48 sampled pixels
    G_dev = iht.adjoint_batched(pool[0], yhat).cpu().numpy()
    cols = np.sort(rng.choice(p.N, 48, replace=False))
    A0 = _radio_cols(p, 0, c_ref, cols)
    for b in rng.choice(B, 8, replace=False):
        y_codes, c_y = OQ.quantize_vector(Y[b], p.b_y, 0, p.seed, snapshot=int(b))
        y_hat = OQ.dequantize(y_codes, c_y, p.b_y, 0)
        assert rel_l2(yhat[b].cpu().numpy(), stack(y_hat, p.M)) < 1e-6
        g_ref = OI.adjoint(A0, y_hat)
        assert rel_l2(G_dev[b, cols], g_ref) < 1e-3                      # tensor-core path bar
    # forward over each snapshot's true support (s = 64 columns), copy 1
    xi = np.stack([np.asarray(x, np.int32) for x in p.meta["batch_x_idx"]])
    xv = np.stack([np.asarray(v, np.float32) for v in p.meta["batch_x_val"]])
    nz = np.full(B, p.s, np.int32)
    R = iht.forward_batched(pool[1], _to_dev(xi), _to_dev(xv), _to_dev(nz), yhat).cpu().numpy()
    for b in rng.choice(B, 4, replace=False):
        F1 = _radio_cols(p, 1, c_ref, xi[b])
        y_codes, c_y = OQ.quantize_vector(Y[b], p.b_y, 0, p.seed, snapshot=int(b))
        r_ref = OI.forward(F1, np.arange(p.s), xv[b].astype(np.float64), OQ.dequantize(y_codes, c_y, p.b_y, 0))
        assert rel_l2(unstack(R[b], p.M, 2), r_ref) < TOL
    # exact per-snapshot top-64 over N = 65536 on the fp32 a the kernel sees
    mu = np.float32(p.mu)
    zero = np.zeros((B, p.s), np.int32)
    oi, ov, on = iht.threshold_batched(_to_dev(zero), _to_dev(zero.astype(np.float32)), _to_dev(np.zeros(B, np.int32)),
                                       _to_dev(G_dev), float(mu), p.s)
    oi, ov, on = oi.cpu().numpy(), ov.cpu().numpy(), on.cpu().numpy()
    for b in range(B):
        a32 = (mu * G_dev[b]).astype(np.float32)
        ri, rv = OI.hard_threshold(a32.astype(np.float64), p.s)
        assert oi[b, :on[b]].tolist() == ri.tolist()
        np.testing.assert_array_equal(ov[b, :on[b]], rv.astype(np.float32))


def test_config3_single_snapshot_teacher_forced(config5):
    """Config 3 = snapshot 0 of config 5's problem through the single-observation path: the
    int8-MMA GEMV adjoint of the same copy agrees with the oracle on sampled pixels."""
    p, pool, c = config5
    c_ref = OQ.scale_c(p.phi)
    y0 = np.ascontiguousarray(p.meta["batch_y"][:, 0])
    yd = _to_dev(y0)
    yhat, _ = iht.quantize_vec(yd, p.b_y, 0, p.seed, iht.absmax(yd))
    g = iht.adjoint(pool[0], yhat).cpu().numpy()
    rng = np.random.default_rng(33)
    cols = np.sort(rng.choice(p.N, 48, replace=False))
    y_codes, c_y = OQ.quantize_vector(y0, p.b_y, 0, p.seed)
    g_ref = OI.adjoint(_radio_cols(p, 0, c_ref, cols), OQ.dequantize(y_codes, c_y, p.b_y, 0))
    assert rel_l2(g[cols], g_ref) < TOL
