"""Pins for oracle/quantize.py against what the paper and arithmetic fix.

Sec. 3 "Quantization", supp. Lemma 3, SPEC quantize
examples.  None of these re-types the oracle's formula: they check
levels, bracketing, exact round trips, the probability law and the error bound.
"""
import numpy as np
import pytest

from oracle import quantize as Q

SEED = 0x5EED_1802_4907


def _levels(c, bits, mode=0):
    L = Q.num_levels(bits, mode)
    return np.array([-c + 2.0 * c * i / (L - 1) for i in range(L)])


def test_num_levels():
    assert [Q.num_levels(b) for b in (2, 4, 8)] == [4, 16, 256]           # l = 2^b
    assert [Q.num_levels(b, 1) for b in (2, 4, 8)] == [3, 9, 129]         # 2^{b-1}+1


def test_worked_example_c3_b2():
    """SURVEY 8(c) worked example: b=2, c=3 -> levels {-3,-1,1,3}; every fp32 op exact."""
    v = np.array([3.0, -3.0, 1.0, -1.0], dtype=np.float32)
    # on-grid values are reproduced exactly whatever the uniforms
    for copy in range(20):
        codes, c = Q.quantize_matrix(v[None, :], 2, 0, SEED, copy, c=np.float32(3.0))
        assert c == 3.0
        vals = Q.dequantize(codes, c, 2, 0)[0]
        np.testing.assert_array_equal(vals, v.astype(np.float64))
    # v = 0 -> -1 or +1 with probability 1/2 each (S:123 at unit scale)
    n = 200_000
    codes, _ = Q.quantize_matrix(np.zeros((n, 1), np.float32), 2, 0, SEED, 0, c=np.float32(3.0))
    vals = Q.dequantize(codes, 3.0, 2, 0)[:, 0]
    assert set(np.unique(vals)) == {-1.0, 1.0}
    frac = np.mean(vals == 1.0)
    assert abs(frac - 0.5) < 4 * np.sqrt(0.25 / n)
    # v = 0.5 -> 1 w.p. 3/4, -1 w.p. 1/4 (P(l_i) = (l_{i+1} - v)/(l_{i+1} - l_i))
    codes, _ = Q.quantize_matrix(np.full((n, 1), 0.5, np.float32), 2, 0, SEED, 1, c=np.float32(3.0))
    vals = Q.dequantize(codes, 3.0, 2, 0)[:, 0]
    assert set(np.unique(vals)) == {-1.0, 1.0}
    frac = np.mean(vals == 1.0)
    assert abs(frac - 0.75) < 4 * np.sqrt(0.75 * 0.25 / n)
    # v = 2 -> 1 or 3 w.p. 1/2
    codes, _ = Q.quantize_matrix(np.full((n, 1), 2.0, np.float32), 2, 0, SEED, 2, c=np.float32(3.0))
    vals = Q.dequantize(codes, 3.0, 2, 0)[:, 0]
    assert set(np.unique(vals)) == {1.0, 3.0}


def test_spec_unit_scale_examples():
    """v = 1.0 with c = 1, b = 2 -> level +1 always; endpoints round-trip."""
    v = np.array([[1.0, -1.0]], dtype=np.float32)
    for copy in range(10):
        codes, c = Q.quantize_matrix(v, 2, 0, SEED, copy)
        assert c == 1.0
        np.testing.assert_array_equal(Q.dequantize(codes, c, 2, 0), v.astype(np.float64))


@pytest.mark.parametrize("bits,mode", [(2, 0), (4, 0), (8, 0), (3, 1), (4, 1), (8, 1)])
def test_on_grid_fixture_round_trips(bits, mode):
    """With c = L-1 the levels are the integers 2i-(L-1) and sf = 1/2: every level
    is reproduced exactly (values exactly on a level are deterministic, reading c5)."""
    L = Q.num_levels(bits, mode)
    lv = np.array([2 * i - (L - 1) for i in range(L)], dtype=np.float32)
    phi = np.tile(lv, (7, 1))
    codes, c = Q.quantize_matrix(phi, bits, mode, SEED, 3)
    assert c == L - 1
    np.testing.assert_array_equal(codes[0], np.tile(np.arange(L), (7, 1)))
    np.testing.assert_array_equal(Q.dequantize(codes, c, bits, mode), phi.astype(np.float64))


@pytest.mark.parametrize("bits,mode", [(2, 0), (4, 0), (8, 0), (4, 1)])
def test_bracketing_and_grid(bits, mode):
    """Q(v) is one of the two levels bracketing v and always on the grid."""
    rng = np.random.default_rng(7)
    phi = rng.standard_normal((64, 96)).astype(np.float32)
    codes, c = Q.quantize_matrix(phi, bits, mode, SEED, 11)
    L = Q.num_levels(bits, mode)
    assert codes.max() <= L - 1
    lv = _levels(float(c), bits, mode)
    vals = Q.dequantize(codes, c, bits, mode)
    np.testing.assert_allclose(vals, lv[codes[0]], rtol=0, atol=1e-12 * float(c))
    t = (phi.astype(np.float64) + float(c)) * (L - 1) / (2.0 * float(c))
    eps = 1e-5 * (L - 1)
    lo = np.floor(t - eps)
    hi = np.ceil(t + eps)
    assert np.all(codes[0] >= lo) and np.all(codes[0] <= hi)
    # away from levels the code is exactly floor or ceil of the exact t
    frac = t - np.floor(t)
    far = (frac > 1e-4) & (frac < 1 - 1e-4)
    k = codes[0][far]
    assert np.all((k == np.floor(t[far])) | (k == np.ceil(t[far])))


@pytest.mark.parametrize("bits", [2, 4, 8])
@pytest.mark.parametrize("vfrac", [0.37, -0.9, 0.0])
def test_unbiased_monte_carlo(bits, vfrac):
    """E[Q(v)] = v within 4 standard errors over 10^6 draws.
    The draws vary the element index (and hence the Philox counter)."""
    c = np.float32(1.7)
    v = np.float32(vfrac * float(c))
    n = 1_000_000
    vec = np.full(n, v, dtype=np.float32)
    vec[0] = c          # fixes the scale c of the tensor
    codes, cc = Q.quantize_vector(vec, bits, 0, SEED + bits)
    assert cc == c
    vals = Q.dequantize(codes, cc, bits, 0)[1:]
    L = 1 << bits
    spacing = 2.0 * float(c) / (L - 1)
    t = (float(v) + float(c)) / spacing
    p = t - np.floor(t)
    se = spacing * np.sqrt(max(p * (1 - p), 1e-300) / (n - 1))
    assert abs(vals.mean() - float(v)) <= 4 * se + 1e-12


@pytest.mark.parametrize("bits", [2, 4, 8])
def test_upper_probability_law(bits):
    """P(upper level) = p = t - floor(t) for many distinct p at once:
    binomial z-test per p-bucket."""
    rng = np.random.default_rng(bits)
    c = np.float32(1.0)
    vals = rng.uniform(-0.99, 0.99, size=64).astype(np.float32)
    reps = 20_000
    phi = np.tile(vals, (reps, 1))
    phi[0, 0] = 1.0
    codes, cc = Q.quantize_matrix(phi, bits, 0, SEED, 5, c=c)
    L = 1 << bits
    t = (vals.astype(np.float64) + 1.0) * (L - 1) / 2.0
    p = t - np.floor(t)
    up = (codes[0][1:] == np.floor(t)[None, :] + 1).mean(axis=0)
    z = (up - p) / np.sqrt(np.maximum(p * (1 - p), 1e-12) / (reps - 1))
    assert np.all(np.abs(z[1:]) < 5.0)


@pytest.mark.parametrize("M", [16, 900])
@pytest.mark.parametrize("bits", [2, 4, 8])
def test_lemma3_bound(M, bits):
    """Supp. Lemma 3: E||Q(v,b) - v||_2 <= c_v sqrt(M) / 2^{b-1}."""
    rng = np.random.default_rng(M + bits)
    errs, bounds = [], []
    for trial in range(100):
        v = rng.standard_normal(M).astype(np.float32)
        codes, c = Q.quantize_vector(v, bits, 0, SEED + trial)
        errs.append(np.linalg.norm(Q.dequantize(codes, c, bits, 0) - v.astype(np.float64)))
        bounds.append(Q.lemma3_bound(c, M, bits))
        # per component the error is below one level spacing 2c/(L-1)
        assert np.max(np.abs(Q.dequantize(codes, c, bits, 0) - v)) <= 2 * float(c) / ((1 << bits) - 1) * (1 + 1e-6)
    assert np.mean(errs) <= np.mean(bounds)
    # SPEC S:149-150 numeric values of the bound
    assert Q.lemma3_bound(1.0, 4, 2) == pytest.approx(1.0)
    assert Q.lemma3_bound(1.0, 900, 8) == pytest.approx(0.234375)


def test_complex_is_two_independent_planes():
    """Complex Phi: re and im quantised independently with the shared scale."""
    rng = np.random.default_rng(3)
    z = (rng.standard_normal((16, 24)) + 1j * rng.standard_normal((16, 24))).astype(np.complex64)
    codes, c = Q.quantize_matrix(z, 4, 0, SEED, 2)
    assert c == max(np.abs(z.real).max(), np.abs(z.imag).max())
    u_re = Q.uniforms24(np.arange(16, dtype=np.uint64)[:, None], np.arange(24, dtype=np.uint64)[None, :],
                        2, 0, Q.TAG_PHI, SEED)
    u_im = Q.uniforms24(np.arange(16, dtype=np.uint64)[:, None], np.arange(24, dtype=np.uint64)[None, :],
                        2, 1, Q.TAG_PHI, SEED)
    assert not np.array_equal(u_re, u_im)
    np.testing.assert_array_equal(codes[0], Q.quantize_component(z.real, c, 4, 0, u_re))
    np.testing.assert_array_equal(codes[1], Q.quantize_component(z.imag, c, 4, 0, u_im))


def test_block_independence_and_determinism():
    """Codes depend only on global (m, n): a block equals the same block of the whole."""
    rng = np.random.default_rng(4)
    phi = rng.standard_normal((40, 37)).astype(np.float32)
    full, c = Q.quantize_matrix(phi, 2, 0, SEED, 9)
    blk, _ = Q.quantize_matrix(phi[13:31, 5:34], 2, 0, SEED, 9, c=c, row_offset=13, col_offset=5)
    np.testing.assert_array_equal(full[:, 13:31, 5:34], blk)
    again, _ = Q.quantize_matrix(phi, 2, 0, SEED, 9)
    np.testing.assert_array_equal(full, again)
    other, _ = Q.quantize_matrix(phi, 2, 0, SEED, 10)
    assert not np.array_equal(full, other)


def test_zero_tensor():
    """c = 0: all-zero quantisation (S:127, S:140 reading 7 of the Q-contract)."""
    codes, c = Q.quantize_matrix(np.zeros((3, 5), np.float32), 4, 0, SEED, 0)
    assert c == 0.0
    assert np.all(Q.dequantize(codes, c, 4, 0) == 0.0)
