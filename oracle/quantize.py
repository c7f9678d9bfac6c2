"""Stochastic quantizer Q_b -- oracle (TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

Paper, Sec. 3 "Quantization": a value v on [-1, 1] that falls in
[l_i, l_{i+1}] of l = 2^b equally spaced levels (l_1 = -1, l_l = +1) is mapped to
l_i with probability (l_{i+1} - v)/(l_{i+1} - l_i), else to l_{i+1}; the map is
unbiased, E[Q_b(v)] = v.  Supp. Lemma 3 scales a vector by
c_v = max |v_j| ("the maximum value of the components of v in magnitude").
The odd-level remark gives 2^{b-1}+1 levels ("level_mode 1").

This file writes out the fp32 Q-contract of DESIGN.md ("Q-contract"), the
reading (c3, c4, c5) that makes every code reproducible bit for bit:

  L      = 2^b (mode 0) or 2^{b-1}+1 (mode 1)                    [P:300, P:689]
  c      = max over all components |Re|, |Im| of the tensor        [P:686, c3]
  sf     = fl32( fl32(L-1) / fl32(2c) )       (sf = 0 when c = 0)
  t      = fl32( fl32(v + c) * sf ), clamped to [0, L-1]
  i      = floor(t);  code = L-1 if i = L-1, else
  p      = t - i  (exact),  u = (w >> 8) * 2^-24,  code = i + (u < p)
  value  = sigma * (2*code - (L-1)),  sigma = c/(L-1)               [levels on [-c, c]]

w is Philox4x32-10 output word (n & 3) for counter
(n >> 2, m, copy_id, (plane << 8) | tag) and key (lo32(seed), hi32(seed)),
with (m, n) the GLOBAL logical row/column of the component; a vector uses
n = 0, m = element index.  tag 0 = Phi, tag 1 = y.  Every fp32 operation is a
separate IEEE round-to-nearest-even numpy float32 operation (no fused
multiply-add).  The upper level is taken when u < p, so
P(l_i) = 1 - p = (l_{i+1} - v)/(l_{i+1} - l_i) exactly as P:303 states, up to
the 24-bit resolution of u (P(upper) = ceil(p 2^24)/2^24).
"""
import numpy as np

from .philox import philox4x32_10

TAG_PHI = 0
TAG_Y = 1


def num_levels(bits, level_mode=0):
    """l = 2^b levels or 2^{b-1}+1 odd levels."""
    if level_mode == 0:
        return 1 << bits
    if level_mode == 1:
        return (1 << (bits - 1)) + 1
    raise ValueError("level_mode must be 0 or 1")


def scale_c(tensor):
    """c = max |component| over the whole tensor, real and imaginary parts pooled
    ("maximum value of the components ... in magnitude"; reading c3).
    Returned as float32 (an fp32 max is exact)."""
    a = np.asarray(tensor)
    if np.iscomplexobj(a):
        a32 = a.astype(np.complex64)
        m = max(np.abs(a32.real).max(initial=0.0), np.abs(a32.imag).max(initial=0.0))
    else:
        m = np.abs(a.astype(np.float32)).max(initial=0.0)
    return np.float32(m)


def uniforms24(m, n, copy_id, plane, tag, seed):
    """u = (w >> 8) * 2^-24 for element (m, n): the 24-bit uniform of the Q-contract."""
    m = np.asarray(m, dtype=np.uint64)
    n = np.asarray(n, dtype=np.uint64)
    m, n = np.broadcast_arrays(m, n)
    k0 = int(seed) & 0xFFFFFFFF
    k1 = (int(seed) >> 32) & 0xFFFFFFFF
    w = philox4x32_10(n >> np.uint64(2), m, copy_id, (plane << 8) | tag, k0, k1)
    sel = (n & np.uint64(3)).astype(np.int64)
    word = np.choose(sel, w)
    # (w >> 8) < 2^24 is exact in float32; times 2^-24 is an exact power-of-two scaling.
    return (word >> np.uint32(8)).astype(np.float32) * np.float32(2.0 ** -24)


def uniforms24_block(row0, rows, col0, cols, copy_id, plane, tag, seed):
    """uniforms24 for the block of global rows [row0, row0+rows) x columns
    [col0, col0+cols): one Philox call per (m, n >> 2), its four words serving
    columns 4(n>>2) .. 4(n>>2)+3 (identical values to uniforms24)."""
    g0 = col0 >> 2
    g1 = (col0 + cols + 3) >> 2
    m = np.arange(row0, row0 + rows, dtype=np.uint64)[:, None]
    g = np.arange(g0, g1, dtype=np.uint64)[None, :]
    k0 = int(seed) & 0xFFFFFFFF
    k1 = (int(seed) >> 32) & 0xFFFFFFFF
    w = philox4x32_10(g, m, copy_id, (plane << 8) | tag, k0, k1)
    words = np.stack(w, axis=-1).reshape(rows, 4 * (g1 - g0))     # column 4g + j <- word j
    off = col0 - 4 * g0
    words = words[:, off:off + cols]
    return (words >> np.uint32(8)).astype(np.float32) * np.float32(2.0 ** -24)


def quantize_component(v, c, bits, level_mode, u):
    """Q-contract rounding of fp32 components v (any shape) given uniforms u.

    Follows Sec. 3 "Quantization" with the fp32 operation sequence
    of the Q-contract.  Returns uint8/uint16 codes in [0, L-1].
    """
    L = num_levels(bits, level_mode)
    v = np.asarray(v, dtype=np.float32)
    c = np.float32(c)
    if c == np.float32(0.0):
        sf = np.float32(0.0)
    else:
        sf = np.float32(np.float32(L - 1) / np.float32(np.float32(2.0) * c))
    t = np.float32(1.0) * (v + c)              # fl32(v + c)
    t = (t * sf).astype(np.float32)             # fl32(t * sf)
    t = np.clip(t, np.float32(0.0), np.float32(L - 1)).astype(np.float32)
    i = np.floor(t).astype(np.int64)
    p = (t - i.astype(np.float32)).astype(np.float32)   # exact (Sterbenz)
    up = (np.asarray(u, dtype=np.float32) < p).astype(np.int64)
    code = np.where(i >= L - 1, L - 1, i + up)
    dtype = np.uint8 if L <= 256 else np.uint16
    return code.astype(dtype)


def quantize_matrix(phi, bits, level_mode, seed, copy_id, c=None, row_offset=0, col_offset=0):
    """Quantize an M x N matrix (float32, or complex64 = two planes) into codes.

    Returns (codes, c) with codes of shape (planes, M, N).  Row / column offsets
    give the global logical indices of the block (codes depend only on global
    indices, so a block quantizes identically to the same block of the whole).
    """
    phi = np.asarray(phi)
    if c is None:
        c = scale_c(phi)
    M, N = phi.shape
    if np.iscomplexobj(phi):
        planes = [phi.real.astype(np.float32), phi.imag.astype(np.float32)]
    else:
        planes = [phi.astype(np.float32)]
    out = []
    for plane, comp in enumerate(planes):
        u = uniforms24_block(row_offset, M, col_offset, N, copy_id, plane, TAG_PHI, seed)
        out.append(quantize_component(comp, c, bits, level_mode, u))
    return np.stack(out), np.float32(c)


def quantize_vector(y, bits, level_mode, seed, c=None, snapshot=0):
    """Quantize the observation vector once (Alg. 1 input y-hat):
    n = snapshot, m = element index, copy 0, tag 1.  A batch of B observations sharing
    Phi (BASELINE config 5) is the matrix Y = [y_0 .. y_{B-1}], observation b being its
    column n = b; a single observation is snapshot 0.  Returns (codes (planes, M), c)."""
    y = np.asarray(y)
    if c is None:
        c = scale_c(y)
    M = y.shape[0]
    m = np.arange(M, dtype=np.uint64)
    n = np.full(M, snapshot, dtype=np.uint64)
    if np.iscomplexobj(y):
        planes = [y.real.astype(np.float32), y.imag.astype(np.float32)]
    else:
        planes = [y.astype(np.float32)]
    out = []
    for plane, comp in enumerate(planes):
        u = uniforms24(m, n, 0, plane, TAG_Y, seed)
        out.append(quantize_component(comp, c, bits, level_mode, u))
    return np.stack(out), np.float32(c)


def dequantize(codes, c, bits, level_mode):
    """value = sigma * (2 code - (L-1)), sigma = c/(L-1), in float64; planes are
    recombined into a complex array when there are two (re, im)."""
    L = num_levels(bits, level_mode)
    sigma = float(c) / (L - 1)
    q = 2.0 * codes.astype(np.float64) - (L - 1)
    vals = sigma * q
    if vals.shape[0] == 2:
        return vals[0] + 1j * vals[1]
    return vals[0]


def lemma3_bound(c, M, bits):
    """Supp. Lemma 3: E||Q(v,b) - v||_2 <= c sqrt(M) / 2^{b-1}."""
    return float(c) * np.sqrt(M) / 2.0 ** (bits - 1)
