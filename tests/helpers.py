"""Test-side helpers: layout unpacking and comparison metrics (no method arithmetic)."""
import numpy as np


def rows_pad(rows):
    return (rows + 255) // 256 * 256


def detile(codes_u8, cols, sb):
    """Tiled copy bytes -> per-column strips (cols, sb) (iht.h: 16-column tiles, 64-byte pieces)."""
    ntiles = (cols + 15) // 16
    arr = np.asarray(codes_u8, dtype=np.uint8)[: ntiles * 16 * sb].reshape(ntiles, sb // 64, 16, 64)
    return arr.transpose(0, 2, 1, 3).reshape(ntiles * 16, sb)[:cols]


def unpack_strips(codes_u8, rows, cols, planes, bits):
    """Copy bytes -> codes array (planes, rows, cols) (iht.h layout)."""
    rp = rows_pad(rows)
    sb = planes * rp * bits // 8
    strips = detile(codes_u8, cols, sb)
    out = np.empty((planes, rows, cols), dtype=np.uint8)
    per_byte = 8 // bits
    mask = (1 << bits) - 1
    for p in range(planes):
        seg = strips[:, p * rp * bits // 8:(p + 1) * rp * bits // 8]        # (cols, rp*bits/8)
        vals = np.empty((cols, rp), dtype=np.uint8)
        for k in range(per_byte):
            vals[:, k::per_byte] = (seg >> (k * bits)) & mask
        out[p] = vals[:, :rows].T
    return out


def pad_rows_of_strips(codes_u8, rows, cols, planes, bits):
    """The pad rows' codes (must be 0)."""
    rp = rows_pad(rows)
    sb = planes * rp * bits // 8
    strips = detile(codes_u8, cols, sb)
    per_byte = 8 // bits
    mask = (1 << bits) - 1
    pads = []
    for p in range(planes):
        seg = strips[:, p * rp * bits // 8:(p + 1) * rp * bits // 8]
        vals = np.empty((cols, rp), dtype=np.uint8)
        for k in range(per_byte):
            vals[:, k::per_byte] = (seg >> (k * bits)) & mask
        pads.append(vals[:, rows:])
    return np.concatenate(pads, axis=1) if pads else np.zeros((cols, 0))


def stack(vec, rows):
    """Complex or real length-rows vector -> stacked real vector (planes * rows_pad), pads 0."""
    vec = np.asarray(vec)
    rp = rows_pad(rows)
    if np.iscomplexobj(vec):
        out = np.zeros(2 * rp)
        out[:rows] = vec.real
        out[rp:rp + rows] = vec.imag
    else:
        out = np.zeros(rp)
        out[:rows] = vec
    return out


def unstack(stacked, rows, planes):
    rp = rows_pad(rows)
    stacked = np.asarray(stacked, dtype=np.float64)
    if planes == 2:
        return stacked[:rows] + 1j * stacked[rp:rp + rows]
    return stacked[:rows]


def rel_l2(got, ref, floor=0.0):
    got = np.asarray(got, dtype=np.complex128 if np.iscomplexobj(got) or np.iscomplexobj(ref) else np.float64)
    ref = np.asarray(ref, dtype=got.dtype)
    den = max(np.linalg.norm(ref), floor)
    if den == 0.0:
        return float(np.linalg.norm(got))
    return float(np.linalg.norm(got - ref) / den)


def dense(idx, val, N):
    x = np.zeros(N)
    x[np.asarray(idx, dtype=np.int64)] = val
    return x


def near_tie(rec_a, margin, s, rel=1e-5):
    """The parity rule's near-tie test: the oracle's gap between the s-th and
    (s+1)-th largest |a| is at most rel * |a|_(s), so fp32 and fp64 may legitimately pick
    different supports from here on."""
    mag = np.sort(np.abs(np.asarray(rec_a)))[::-1]
    if s <= 0 or mag.size == 0:
        return False
    kth = mag[min(s, mag.size) - 1]
    return not margin > rel * max(kth, 1e-30)


def check_trajectory(trace, idx, val, nnz, s, tol):
    """Free-running comparison of a solver trace with the oracle's records: every iteration
    before the oracle's first near-tie must have the identical support and x within `tol`
    relative l2 (no escape).  idx / val: [n_iter][s], nnz: [n_iter] (row n = x after
    iteration n+1).  Returns the number of compared iterations (len(trace) = no near-tie)."""
    idx, val, nnz = np.asarray(idx), np.asarray(val), np.asarray(nnz)
    for n, rec in enumerate(trace):
        if near_tie(rec.a, rec.margin, s):
            return n
        k = int(nnz[n])
        assert idx[n, :k].tolist() == list(rec.x_idx), \
            f"iteration {rec.n}: support differs from the oracle (margin {rec.margin:.3e})"
        err = rel_l2(val[n, :k], rec.x_val, floor=1e-30)
        assert err <= tol, f"iteration {rec.n}: x relative l2 error {err:.3e} > {tol}"
    return len(trace)
