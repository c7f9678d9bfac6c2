"""Input generators (workloads/): determinism, random access, distributions."""
import numpy as np

from workloads import gen as G


def test_counter_gaussian_block_access_and_moments():
    key = G.derive_key(99, 1)
    full = G.gaussian_block(key, 300, 0, 200, 0, 300, 0.5)
    blk = G.gaussian_block(key, 300, 37, 50, 101, 77, 0.5)
    np.testing.assert_array_equal(full[37:87, 101:178], blk)
    cols = G.gaussian_columns(key, 300, 10, 20, [5, 299, 0], 0.5)
    np.testing.assert_array_equal(cols, full[10:30][:, [5, 299, 0]])
    assert abs(full.mean()) < 0.01
    assert abs(full.std() - 0.5) < 0.01
    # Irwin-Hall(12) is bounded at 6 sd
    assert np.abs(full).max() <= 6 * 0.5 + 1e-6
    # exact integer construction: value * 2*sqrt(65536^2-1)/sd is (close to) an even-offset integer
    z = G.gauss_int(key, np.arange(1000, dtype=np.uint64))
    assert np.all(np.abs(z) < 2 ** 20) and np.all(z % 2 == 12 * 65535 % 2)


def test_gaussian_problem_consistency():
    p = G.gaussian_problem(64, 200, 5, cfg_id=77, noise_sd=0.0)
    assert p.phi.dtype == np.float32 and p.y.dtype == np.float32
    x = np.zeros(200)
    x[p.x_idx] = p.x_val
    np.testing.assert_allclose(p.y, p.phi.astype(np.float64) @ x, rtol=1e-5, atol=1e-6)
    q = G.gaussian_problem(64, 200, 5, cfg_id=77, noise_sd=0.0, materialize=False)
    np.testing.assert_array_equal(q.y, p.y)
    np.testing.assert_array_equal(q.phi_rows(10, 7), p.phi[10:17])
    np.testing.assert_array_equal(q.phi_cols([3, 9], 5, 4), p.phi[5:9][:, [3, 9]])


def test_radio_generator_properties():
    """Unit-modulus entries; zero-baseline (autocorrelation) rows are all ones;
    M = A^2 (reading c16)."""
    p = G.radio_problem(cfg_id=3, A=6, grid=16, n_src=4, n_iter=5)
    assert p.phi.shape == (36, 256) and p.complex
    np.testing.assert_allclose(np.abs(p.phi), 1.0, rtol=1e-6)
    for i in range(6):
        np.testing.assert_allclose(p.phi[i * 6 + i], 1.0 + 0j, atol=1e-7)
    # Hermitian symmetry of baselines: row (i,j) = conj(row (j,i))
    np.testing.assert_allclose(p.phi[1 * 6 + 2], np.conj(p.phi[2 * 6 + 1]), atol=1e-6)
    l, m = p.meta["l"], p.meta["m"]
    assert np.all(l[p.x_idx] ** 2 + m[p.x_idx] ** 2 < 1.0)
    assert np.all(p.x_val > 0)


def test_config_steps_follow_reading_c9():
    """Fixed steps of the BASELINE configs (DESIGN reading c9): config 1 and 4 the stated
    mu = 1, config 2 mu = 1/4 (mu = 1 diverges at 2 bits), radio mu = 1/(10 M)."""
    assert G.CONFIGS[1].get("mu", 1.0) == 1.0 and G.CONFIGS[4].get("mu", 1.0) == 1.0
    assert G.CONFIGS[2]["mu"] == 0.25
    p = G.radio_problem(cfg_id=99, A=6, grid=16, n_src=3, n_iter=2, K=2)
    assert p.mu == 0.1 / p.M
    q = G.gaussian_problem(64, 128, 4, cfg_id=98, n_iter=2, mu=0.25, K=2)
    assert q.mu == 0.25


def test_config6_is_the_paper_imaging_shape_at_0dB():
    """Config 6 = the paper's imaging experiment shape: y in C^900, Phi-hat in
    C^{900 x 65536} (30 antennas, 256 x 256 pixels), 30 sources, SNR 0 dB at the antenna level,
    10 log10(||Phi x||^2 / ||e||^2) = 0 -- here within the chi-square spread of 900 complex
    noise draws (+-0.3 dB, > 4 standard deviations)."""
    c = G.CONFIGS[6]
    assert (c["A"] ** 2, c["grid"] ** 2, c["n_src"], c["b_phi"], c["b_y"]) == (900, 65536, 30, 2, 8)
    p = G.config_problem(6, K=2)
    assert (p.M, p.N, p.s, p.complex) == (900, 65536, 30, True)
    vis = p.phi[:, p.x_idx].astype(np.complex128) @ p.x_val
    e = p.y.astype(np.complex128) - vis
    snr_db = 10 * np.log10(np.sum(np.abs(vis) ** 2) / np.sum(np.abs(e) ** 2))
    assert abs(snr_db) < 0.3, snr_db
    assert 15e6 <= 299792458.0 / p.meta["wavelength"] <= 80e6      # the low band
