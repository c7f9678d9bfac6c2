"""Seeded synthetic inputs for BASELINE.json's configs (no method arithmetic here).

Recipe:

* Gaussian entries come from a counter-based generator so that any block of a
  65536 x 262144 matrix can be regenerated independently, on the host (numpy,
  here) or on the GPU (workloads/csrc/gen.cu), bit for bit:
      h_j   = mix64(key + (3*idx + j + 1) * 0x9E3779B97F4A7C15),  j = 0, 1, 2
      S     = sum of the twelve 16-bit fields of h_0, h_1, h_2      (Irwin-Hall(12))
      z     = 2*S - 12*65535                 (an exact integer, |z| < 2^20)
      value = fl32( fl32(z) * scale32 ),  scale32 = fl32(sd / (2*sqrt(65536^2 - 1)))
  so value has mean 0 and standard deviation sd (up to the 16-bit grid), with
  idx = m * N + n the global row-major index.  Irwin-Hall(12) stands in for
  N(0, sd^2): it is bounded at +-6 sd; DESIGN.md states this.
* Support positions and values of x, antenna positions and the noise e are drawn
  on the host with numpy's PCG64 seeded by SeedSequence([1802, 4907, cfg_id]).
* y = Phi x + e is accumulated in float64 over the fp32 Phi entries and stored
  as fp32 (complex64 for radio); the same fp32 (Phi, y) feed the oracle and the
  CUDA path.
"""
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

GOLDEN = 0x9E3779B97F4A7C15
MASK64 = (1 << 64) - 1


def mix64(z):
    """SplitMix64 finaliser on uint64 numpy arrays (wrapping arithmetic)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def derive_key(cfg_id, stream):
    """64-bit key of one generator stream (1 = Phi) of one config."""
    base = ((1802 << 48) ^ (4907 << 32) ^ (int(cfg_id) << 8) ^ int(stream)) & MASK64
    return int(mix64(np.array([base], dtype=np.uint64))[0])


def counter_hash(key, ctr):
    """mix64(key + (ctr + 1) * GOLDEN) for uint64 counters ctr."""
    ctr = np.asarray(ctr, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(key) + (ctr + np.uint64(1)) * np.uint64(GOLDEN)
    return mix64(z)


def gauss_int(key, idx):
    """The exact integer z = 2*S - 12*65535 of element idx (see module doc)."""
    idx = np.asarray(idx, dtype=np.uint64)
    s = np.zeros(idx.shape, dtype=np.int64)
    for j in range(3):
        h = counter_hash(key, idx * np.uint64(3) + np.uint64(j))
        for f in range(4):
            s += ((h >> np.uint64(16 * f)) & np.uint64(0xFFFF)).astype(np.int64)
    return 2 * s - 12 * 65535


def gauss_scale32(sd):
    """scale32 = fl32(sd / (2 sqrt(65536^2 - 1)))."""
    return np.float32(float(sd) / (2.0 * np.sqrt(65536.0 ** 2 - 1.0)))


def gaussian_block(key, n_total, row0, rows, col0, cols, sd):
    """fp32 block Phi[row0:row0+rows, col0:col0+cols] of the counter-Gaussian matrix
    with n_total columns (global row-major index m * n_total + n)."""
    m = np.arange(row0, row0 + rows, dtype=np.uint64)[:, None]
    n = np.arange(col0, col0 + cols, dtype=np.uint64)[None, :]
    z = gauss_int(key, m * np.uint64(n_total) + n)
    return (z.astype(np.float32) * gauss_scale32(sd)).astype(np.float32)


def gaussian_columns(key, n_total, row0, rows, col_idx, sd):
    """fp32 Phi[row0:row0+rows, col_idx] for an arbitrary list of columns."""
    m = np.arange(row0, row0 + rows, dtype=np.uint64)[:, None]
    n = np.asarray(col_idx, dtype=np.uint64)[None, :]
    z = gauss_int(key, m * np.uint64(n_total) + n)
    return (z.astype(np.float32) * gauss_scale32(sd)).astype(np.float32)


@dataclass
class ProblemSpec:
    """One synthetic CS problem y = Phi x + e plus its solver settings."""
    name: str
    cfg_id: int
    M: int                       # measurements (visibilities)
    N: int                       # unknowns (pixels)
    complex: bool
    s: int
    n_iter: int
    mu: float
    b_phi: int
    b_y: int
    K: int                       # pool of independent quantised copies (reading c6)
    seed: int                    # quantiser seed
    x_idx: np.ndarray
    x_val: np.ndarray
    y: np.ndarray                # fp32 / complex64, length M
    phi: Optional[np.ndarray] = None   # fp32 / complex64 (M, N) when materialised
    phi_key: Optional[int] = None      # counter key for Gaussian Phi (regenerable)
    phi_sd: Optional[float] = None
    meta: dict = field(default_factory=dict)

    @property
    def planes(self):
        return 2 if self.complex else 1

    @property
    def R(self):
        """Stacked real rows (re plane then im plane)."""
        return self.M * self.planes

    def phi_rows(self, row0, rows):
        """Rows [row0, row0+rows) of Phi (regenerated if not materialised)."""
        if self.phi is not None:
            return self.phi[row0:row0 + rows]
        return gaussian_block(self.phi_key, self.N, row0, rows, 0, self.N, self.phi_sd)

    def phi_cols(self, col_idx, row0=0, rows=None):
        rows = self.M - row0 if rows is None else rows
        if self.phi is not None:
            return self.phi[row0:row0 + rows][:, col_idx]
        return gaussian_columns(self.phi_key, self.N, row0, rows, col_idx, self.phi_sd)


def quant_seed(cfg_id):
    return 0x18020490700 + int(cfg_id)


def _rng(cfg_id):
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([1802, 4907, int(cfg_id)])))


def gaussian_problem(M, N, s, *, cfg_id, values="normal", noise_sd=0.01, n_iter=100, mu=1.0,
                     b_phi=4, b_y=8, K=2, materialize=True, name=None, entry_sd=None):
    """Real Gaussian CS (BASELINE configs 1, 2, 4; supp. toy P:1216-1224):
    Phi_mn ~ N(0, 1/M) (counter Irwin-Hall(12) stand-in), x with s nonzeros at
    uniform random positions, values N(0,1) ('normal') or +-1 ('sign'),
    y = Phi x + e, e ~ N(0, noise_sd^2)."""
    key = derive_key(cfg_id, 1)
    sd = 1.0 / np.sqrt(M) if entry_sd is None else entry_sd
    rng = _rng(cfg_id)
    x_idx = np.sort(rng.choice(N, size=s, replace=False)).astype(np.int64)
    if values == "normal":
        x_val = rng.standard_normal(s)
    elif values == "sign":
        x_val = rng.choice(np.array([-1.0, 1.0]), size=s)
    else:
        raise ValueError(values)
    e = noise_sd * rng.standard_normal(M)
    phi = gaussian_block(key, N, 0, M, 0, N, sd) if materialize else None
    # y = Phi x + e, accumulated in float64 over fp32 entries, block-wise by rows
    y = np.empty(M, dtype=np.float64)
    blk = 4096
    for r0 in range(0, M, blk):
        rows = min(blk, M - r0)
        cols = (phi[r0:r0 + rows][:, x_idx] if phi is not None
                else gaussian_columns(key, N, r0, rows, x_idx, sd))
        y[r0:r0 + rows] = cols.astype(np.float64) @ x_val
    y = (y + e).astype(np.float32)
    return ProblemSpec(name or f"gauss-{M}x{N}", cfg_id, M, N, False, s, n_iter, mu, b_phi, b_y,
                       K, quant_seed(cfg_id), x_idx, x_val, y, phi, key, sd)


def radio_antennas(A, radius_m, rng):
    """A antennas uniform in a disc (r = R sqrt(U), theta = 2 pi U')."""
    r = radius_m * np.sqrt(rng.random(A))
    th = 2.0 * np.pi * rng.random(A)
    return np.stack([r * np.cos(th), r * np.sin(th)], axis=1)


def radio_phi(pos, wavelength, grid):
    """Phi_{k,p} = exp(-2 pi i b_k . (l_p, m_p) / lambda) (BASELINE config 3; supp.
    "Formation of Phi", reading c16): b_k = pos_i - pos_j with
    k = i*A + j (autocorrelations kept, M = A^2), pixel p = row*grid + col with
    cell-centred direction cosines l, m in (-1, 1).  float64 -> complex64."""
    A = pos.shape[0]
    b = (pos[:, None, :] - pos[None, :, :]).reshape(A * A, 2)          # k = i*A + j
    centres = -1.0 + (2.0 * np.arange(grid) + 1.0) / grid
    l = np.repeat(centres, grid)          # p = row*grid + col: row -> l
    m = np.tile(centres, grid)            # col -> m
    phi = np.empty((A * A, grid * grid), dtype=np.complex64)
    blk = 256
    for k0 in range(0, A * A, blk):
        bk = b[k0:k0 + blk]
        phase = -2.0 * np.pi * (np.outer(bk[:, 0], l) + np.outer(bk[:, 1], m)) / wavelength
        phi[k0:k0 + blk] = np.exp(1j * phase).astype(np.complex64)
    return phi, l, m


def radio_problem(*, cfg_id, A=48, radius_m=30.0, freq_hz=150e6, grid=256, n_src=64, n_iter=200,
                  b_phi=2, b_y=8, K=2, noise_frac=0.01, name=None, batch=1, mu_scale=0.1, phi_cfg_id=None):
    """Synthetic radio interferometer (BASELINE config 3, batch=64 -> config 5).
    Fixed step mu = mu_scale / M (reading c9): the columns have |Phi_kp| = 1, so 1/M
    normalises them, but the coherent radio Phi diverges at 1/M and 1/4M (|x| -> inf,
    scripts/step_study.py); 1/10 M stays bounded.
    Sources: n_src pixels drawn without replacement among pixels with
    l^2 + m^2 < 1 (reading c19), log-normal(0,1) fluxes; complex noise
    e = (sigma/sqrt 2)(n1 + i n2), sigma = noise_frac * rms visibility (c17).
    phi_cfg_id: take the antenna layout (hence Phi) of that config (config 5 = "the config-3
    Phi", BASELINE): its antennas are the first draws of _rng(phi_cfg_id); the skies and noise
    then come from _rng(cfg_id)."""
    rng = _rng(cfg_id)
    wavelength = 299792458.0 / freq_hz
    if phi_cfg_id is None or phi_cfg_id == cfg_id:
        pos = radio_antennas(A, radius_m, rng)
    else:
        pos = radio_antennas(A, radius_m, _rng(phi_cfg_id))
    phi, l, m = radio_phi(pos, wavelength, grid)
    inside = np.flatnonzero(l * l + m * m < 1.0)
    xs, vs, ys = [], [], []
    for _ in range(batch):
        x_idx = np.sort(rng.choice(inside, size=n_src, replace=False)).astype(np.int64)
        x_val = rng.lognormal(0.0, 1.0, size=n_src)
        vis = phi[:, x_idx].astype(np.complex128) @ x_val
        sigma = noise_frac * np.sqrt(np.mean(np.abs(vis) ** 2))
        e = (sigma / np.sqrt(2.0)) * (rng.standard_normal(A * A) + 1j * rng.standard_normal(A * A))
        xs.append(x_idx)
        vs.append(x_val)
        ys.append((vis + e).astype(np.complex64))
    M = A * A
    spec = ProblemSpec(name or f"radio-{A}ant-{grid}px", cfg_id, M, grid * grid, True, n_src, n_iter,
                       mu_scale / M, b_phi, b_y, K, quant_seed(cfg_id), xs[0], vs[0], ys[0], phi)
    spec.meta.update(antennas=pos, wavelength=wavelength, l=l, m=m)
    if batch > 1:
        spec.meta.update(batch_x_idx=xs, batch_x_val=vs, batch_y=np.stack(ys, axis=1))
    return spec


# BASELINE.json configs (index = cfg_id)
CONFIGS = {
    1: dict(kind="gauss", M=256, N=1024, s=16, values="normal", n_iter=100, b_phi=4, b_y=8),
    # config 2: BASELINE states no step; mu = 1 diverges at 2 bits (|x| -> inf by iteration
    # 195, scripts/step_study.py), mu = 1/4 recovers the support (reading c9)
    2: dict(kind="gauss", M=4096, N=16384, s=128, values="sign", n_iter=200, b_phi=2, b_y=8, mu=0.25),
    3: dict(kind="radio", A=48, grid=256, n_src=64, n_iter=200, b_phi=2, b_y=8),
    4: dict(kind="gauss", M=65536, N=262144, s=1024, values="normal", n_iter=100, b_phi=4, b_y=8),
    5: dict(kind="radio", A=48, grid=256, n_src=64, n_iter=200, b_phi=2, b_y=8, batch=64, phi_cfg_id=3),
    # config 6 (not a BASELINE config): the paper's own imaging experiment shape, P:534 -- 30
    # low-band antennas (M = 900), a 256 x 256 sky (N = 65536), 30 strong sources, SNR 0 dB at
    # the antenna level (||Phi x||^2 = ||e||^2: noise_frac = 1), 2-bit Phi, 8-bit y.  The LOFAR
    # CS302 layout and sky are data we do not have: synthetic antennas in a 40 m-radius disc at
    # 60 MHz (inside the 15-80 MHz band), log-normal fluxes; n* = 200 (not stated).
    # mu = 1/(20 M): at 0 dB the oracle's iterates diverge at 0.1/M and 0.3/M (|x| ~ 1e28 /
    # 1e151 by iteration 199) and stay bounded at 0.05/M (|x| ~ 5.1 from iteration 50 on).
    6: dict(kind="radio", A=30, grid=256, n_src=30, n_iter=200, b_phi=2, b_y=8, noise_frac=1.0,
            radius_m=40.0, freq_hz=60e6, mu_scale=0.05),
}


def config_problem(cfg_id, K=None, materialize=None, b_phi=None):
    """Build BASELINE config cfg_id (1..5; 6 = the paper's P:534 imaging shape).  K defaults to 2 n* where that fits
    (configs 1-3, 5) and 2 for config 4 (reading c6)."""
    c = dict(CONFIGS[cfg_id])
    kind = c.pop("kind")
    if b_phi is not None:
        c["b_phi"] = b_phi
    if kind == "gauss":
        if K is None:
            K = 2 if cfg_id == 4 else 2 * c["n_iter"]
        if materialize is None:
            materialize = cfg_id != 4
        return gaussian_problem(c["M"], c["N"], c["s"], cfg_id=cfg_id, values=c["values"],
                                n_iter=c["n_iter"], mu=c.get("mu", 1.0), b_phi=c["b_phi"], b_y=c["b_y"], K=K,
                                materialize=materialize, name=f"config{cfg_id}")
    if K is None:
        K = 2 * c["n_iter"]
    return radio_problem(cfg_id=cfg_id, A=c["A"], grid=c["grid"], n_src=c["n_src"],
                         n_iter=c["n_iter"], b_phi=c["b_phi"], b_y=c["b_y"], K=K,
                         batch=c.get("batch", 1), name=f"config{cfg_id}", phi_cfg_id=c.get("phi_cfg_id"),
                         **{k: c[k] for k in ("noise_frac", "radius_m", "freq_hz", "mu_scale") if k in c})
