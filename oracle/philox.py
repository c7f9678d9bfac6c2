"""Philox4x32-10 in numpy -- oracle RNG (TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

The paper's CPU code drew its stochastic-rounding randomness from XORShift
(supp. "CPU Implementation Details") and does not fix the generator.
DESIGN.md reading c4 replaces it by the counter-based Philox4x32-10 so that a
code depends only on (seed, copy, tensor, plane, m, n) and can be recomputed
element by element.  Public constants: multipliers M0 = 0xD2511F53,
M1 = 0xCD9E8D57, Weyl key increments W0 = 0x9E3779B9, W1 = 0xBB67AE85;
10 rounds.

Pin: tests/test_oracle_philox.py compares this function with cuRAND's own
``curand_Philox4x32_10`` (CUDA toolkit header, compiled for the host) on a
grid of counters and keys.
"""
import numpy as np

M0 = np.uint64(0xD2511F53)
M1 = np.uint64(0xCD9E8D57)
W0 = 0x9E3779B9
W1 = 0xBB67AE85
_MASK32 = np.uint64(0xFFFFFFFF)
_S32 = np.uint64(32)


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Return the four 32-bit output words for counter (c0,c1,c2,c3), key (k0,k1).

    Arguments are integers or uint32-compatible numpy arrays (broadcast
    together).  One round maps (x0,x1,x2,x3) ->
    (hi(M1*x2) ^ x1 ^ k0, lo(M1*x2), hi(M0*x0) ^ x3 ^ k1, lo(M0*x0)),
    then the key is bumped by (W0, W1); ten rounds in total.
    """
    x0, x1, x2, x3 = (np.asarray(c, dtype=np.uint64) & _MASK32 for c in (c0, c1, c2, c3))
    x0, x1, x2, x3 = np.broadcast_arrays(x0, x1, x2, x3)
    ka = int(k0) & 0xFFFFFFFF
    kb = int(k1) & 0xFFFFFFFF
    for rnd in range(10):
        p0 = M0 * x0          # < 2^64, exact in uint64
        p1 = M1 * x2
        y0 = (p1 >> _S32) ^ x1 ^ np.uint64(ka)
        y1 = p1 & _MASK32
        y2 = (p0 >> _S32) ^ x3 ^ np.uint64(kb)
        y3 = p0 & _MASK32
        x0, x1, x2, x3 = y0, y1, y2, y3
        ka = (ka + W0) & 0xFFFFFFFF
        kb = (kb + W1) & 0xFFFFFFFF
    return tuple(np.asarray(v, dtype=np.uint32) for v in (x0, x1, x2, x3))
