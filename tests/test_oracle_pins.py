"""Pins for the whole oracle procedure, CPU only.

P1 brute-force minimisation of the per-pixel objective (reading C4) on tiny inputs
P2 the closed-form matched filter (Eq. 3) when sparsity/albedo/iterations are off
P3 invariants (positivity, permutations, scaling, homogeneity, beta = 0)
P4 exact recovery on a noiseless separable scene
P5 an independent numpy transcription (oracle/transcription.py)
P6 qualitative sanity on generator scenes
"""
import math

import numpy as np
import pytest
import scipy.linalg
import scipy.optimize

from oracle import transcription
from paper_2003_02978_b200 import synth


def _random_instance(rng, N, B, plume_frac=0.2):
    mu = rng.uniform(2.0, 5.0, size=B)
    A = rng.normal(size=(B, B)) * 0.1
    a = rng.uniform(0.6, 1.4, size=N)
    L = a[:, None] * mu[None, :] + rng.normal(size=(N, B)) @ A.T
    s = -rng.uniform(0.0, 1e-4, size=B)
    m = rng.random(N) < plume_frac
    L[m] *= (1.0 + s[None, :] * rng.uniform(500, 3000, size=m.sum())[:, None])
    return L.astype(np.float32), s.astype(np.float32)


# ---------------------------------------------------------------- P1
@pytest.mark.parametrize("use_sparsity,use_albedo", [(1, 1), (1, 0), (0, 1), (0, 0)])
def test_p1_line16_is_bruteforce_minimiser(oracle_lib, use_sparsity, use_albedo):
    """For every k >= 1 and pixel, alpha^k = argmin_{a>=0} 1/2 d^T (C^k+rho I)^-1 d + r~ w a,
    d = L - r~ a t^k - mu^k, found by dense grid + golden-section search, with the
    oracle's own mu^k, C^k, w = 1/(alpha^{k-1}+eps) and r~ (reading C4)."""
    rng = np.random.default_rng(10 + 2 * use_sparsity + use_albedo)
    checked = 0
    for inst in range(12):
        N, B = int(rng.integers(12, 40)), int(rng.integers(2, 6))
        L, s = _random_instance(rng, N, B)
        n_iter = 3
        alpha, r, rc, dg = oracle_lib.retrieve_column(L, s, n_iter=n_iter, use_sparsity=use_sparsity,
                                                      use_albedo=use_albedo, eps=1e-2, lambda_rel=1e-3,
                                                      diagnostics=True)
        assert rc == 0
        Ld = L.astype(np.float64)
        rt = np.maximum(r, 0.05) if use_albedo else np.ones(N)
        rho = dg["rho"][0]
        sd = s.astype(np.float64)
        for k in range(1, n_iter + 1):
            mu, C = dg["mu"][k], dg["cov"][k]
            t = mu * sd
            # objective evaluated in extended precision so the scalar search is not
            # limited by fp64 rounding of the (flat) quadratic
            Ci = np.linalg.inv(C + rho * np.eye(B)).astype(np.longdouble)
            tl, mul = t.astype(np.longdouble), mu.astype(np.longdouble)
            prev = dg["alpha_hist"][k - 1] if k > 1 else np.maximum(dg["alpha_hist"][0], 0.0)
            w = 1.0 / (prev + 1e-2) if use_sparsity else np.zeros(N)
            for i in range(0, N, 3):
                def J(a):
                    a = np.longdouble(a)
                    d = Ld[i].astype(np.longdouble) - np.longdouble(rt[i]) * a * tl - mul
                    return float(np.longdouble(0.5) * (d @ (Ci @ d)) + np.longdouble(rt[i] * w[i]) * a
                                 - np.longdouble(0.5) * (Ld[i] - mu).astype(np.longdouble) @ (Ci @ (Ld[i] - mu).astype(np.longdouble)))
                grid = np.linspace(0.0, 2.0 * max(5000.0, abs(dg["alpha_hist"][k][i]) * 2), 801)
                vals = np.array([J(a) for a in grid])
                j = int(np.argmin(vals))
                lo, hi = grid[max(j - 1, 0)], grid[min(j + 1, len(grid) - 1)]
                res = scipy.optimize.minimize_scalar(J, bounds=(lo, hi), method="bounded",
                                                     options={"xatol": 1e-10})
                a_bf = res.x if J(res.x) <= J(0.0) else 0.0
                got = dg["alpha_hist"][k][i]
                assert got == pytest.approx(a_bf, rel=1e-6, abs=1e-5), (inst, k, i)
                checked += 1
    assert checked > 100


def test_p1_eq8_literal_gives_half_threshold(oracle_lib):
    """Documents reading C4: minimising Eq. 8 exactly as printed (no 1/2) shrinks by
    w/2, whereas line 16 (implemented) shrinks by w."""
    num, w, r, q = 3.0, 1.0, 1.3, 0.7
    J8 = lambda a: q * r * r * a * a - 2 * r * num * a + r * w * a     # d^T C^-1 d + r w a
    res = scipy.optimize.minimize_scalar(J8, bounds=(0, 100), method="bounded", options={"xatol": 1e-12})
    assert res.x == pytest.approx((num - w / 2) / (r * q), rel=1e-6)
    assert oracle_lib.ista_update(num, w, r, q) == pytest.approx((num - w) / (r * q), rel=1e-14)


# ---------------------------------------------------------------- P2
def test_p2_closed_form_classical_mf(oracle_lib):
    """sparsity off, albedo off, n_iter = 0: Eq. 3 with mu0 = mean, C0 = population
    covariance -- via numpy.cov + scipy.linalg.cho_solve."""
    rng = np.random.default_rng(20)
    for _ in range(5):
        N, B = 300, 8
        L, s = _random_instance(rng, N, B)
        alpha, r, rc = oracle_lib.retrieve_column(L, s, n_iter=0, use_sparsity=0, use_albedo=0)
        assert rc == 0
        Ld = L.astype(np.float64)
        mu = Ld.mean(axis=0)
        C = np.cov(Ld, rowvar=False, bias=True)
        t = mu * s.astype(np.float64)
        z = scipy.linalg.cho_solve(scipy.linalg.cho_factor(C), t)
        ref = (Ld - mu) @ z / (t @ z)
        np.testing.assert_allclose(alpha, ref, rtol=1e-9, atol=1e-9 * np.abs(ref).max())
        np.testing.assert_array_equal(r, 1.0)
        # albedo on, n_iter = 0: Albedo-Only MF (Table I row 2) = Eq. 3 / r_i
        alpha_a, r_a, rc = oracle_lib.retrieve_column(L, s, n_iter=0, use_sparsity=0, use_albedo=1)
        r_ref = Ld @ mu / (mu @ mu)
        np.testing.assert_allclose(r_a, r_ref, rtol=1e-12)
        np.testing.assert_allclose(alpha_a, ref / np.maximum(r_ref, 0.05), rtol=1e-9,
                                   atol=1e-9 * np.abs(ref).max())


# ---------------------------------------------------------------- P3
def _tiny(cols=3, pixels=256, bands=16):
    cfg = synth.scaled(synth.CONFIGS["tiny"], cols=cols, pixels=pixels, bands=bands)
    cube, s, truth = synth.generate(cfg)
    return cube, s, truth


def test_p3_positivity_and_no_negative_zero(oracle_lib):
    cube, s, _ = _tiny()
    for sp in (0, 1):
        alpha, r, st = oracle_lib.retrieve(cube, s, n_iter=5, use_sparsity=sp)
        assert (st == 0).all()
        assert (alpha >= 0).all()
        assert not np.signbit(alpha).any()
    # n_iter = 0 returns the unclamped alpha0 (reading C3)
    alpha0, _, _ = oracle_lib.retrieve(cube, s, n_iter=0)
    assert (alpha0 < 0).any()


def test_p3_pixel_permutation(oracle_lib):
    cube, s, _ = _tiny(cols=2)
    perm = np.random.default_rng(0).permutation(cube.shape[1])
    a, r, _ = oracle_lib.retrieve(cube, s, n_iter=8)
    ap, rp, _ = oracle_lib.retrieve(cube[:, perm], s, n_iter=8)
    np.testing.assert_allclose(ap, a[:, perm], rtol=1e-10, atol=1e-9 * np.abs(a).max())
    np.testing.assert_allclose(rp, r[:, perm], rtol=1e-12)


def test_p3_column_permutation_is_exact(oracle_lib):
    cube, s, _ = _tiny(cols=4)
    perm = np.array([2, 0, 3, 1])
    a, r, _ = oracle_lib.retrieve(cube, s, n_iter=6)
    ap, rp, _ = oracle_lib.retrieve(cube[perm], s, n_iter=6)
    np.testing.assert_array_equal(ap, a[perm])
    np.testing.assert_array_equal(rp, r[perm])


def test_p3_band_permutation(oracle_lib):
    cube, s, _ = _tiny(cols=2)
    perm = np.random.default_rng(1).permutation(cube.shape[2])
    a, r, _ = oracle_lib.retrieve(cube, s, n_iter=6)
    ap, rp, _ = oracle_lib.retrieve(cube[:, :, perm], s[perm], n_iter=6)
    np.testing.assert_allclose(ap, a, rtol=1e-8, atol=1e-8 * np.abs(a).max())
    np.testing.assert_allclose(rp, r, rtol=1e-12)


def test_p3_radiance_scaling(oracle_lib):
    cube, s, _ = _tiny(cols=2)
    a, r, _ = oracle_lib.retrieve(cube, s, n_iter=6, lambda_rel=1e-4)
    # power-of-two scaling is exact in floating point: bitwise identical maps
    a2, r2, _ = oracle_lib.retrieve(cube * np.float32(2.0), s, n_iter=6, lambda_rel=1e-4)
    np.testing.assert_array_equal(a2, a)
    np.testing.assert_array_equal(r2, r)
    a3, r3, _ = oracle_lib.retrieve((cube.astype(np.float64) * 3.0).astype(np.float32), s, n_iter=6,
                                    lambda_rel=1e-4)
    np.testing.assert_allclose(a3, a, rtol=1e-5, atol=1e-5 * np.abs(a).max())


def test_p3_homogeneity_in_s_without_sparsity(oracle_lib):
    """with sparsity off, alpha(c s) = alpha(s) / c."""
    cube, s, _ = _tiny(cols=2)
    a, _, _ = oracle_lib.retrieve(cube, s, n_iter=5, use_sparsity=0)
    a4, _, _ = oracle_lib.retrieve(cube, s * np.float32(4.0), n_iter=5, use_sparsity=0)
    np.testing.assert_allclose(a4 * 4.0, a, rtol=1e-9, atol=1e-9 * np.abs(a).max())


def test_p3_zero_beta_restores_initial_statistics(oracle_lib):
    """all beta = 0 => mu^k = mu0 and C^k = C0 (bitwise). On the separable
    noiseless scene with no plume pixel every projection is exactly 0, so alpha0 = 0
    and beta = r~ alpha = 0 for every pixel."""
    cube, s, _ = synth.noiseless_scene(cols=1, pixels=400, bands=10, frac=0.0)
    a, r, rc, dg = oracle_lib.retrieve_column(cube[0], s, n_iter=3, lambda_rel=1e-3, diagnostics=True)
    assert rc == 0
    assert (dg["alpha_hist"] == 0).all()
    for k in (1, 2, 3):
        np.testing.assert_array_equal(dg["mu"][k], dg["mu"][0])
        np.testing.assert_array_equal(dg["cov"][k], dg["cov"][0])


def test_p3_signal_removal_fixed_point(oracle_lib):
    """statistics after removing the exact generating signal equal those of the
    enhancement-free partition (here via the noiseless scene at convergence)."""
    cube, s, truth = synth.noiseless_scene(cols=1, pixels=300, bands=10)
    a, r, rc, dg = oracle_lib.retrieve_column(cube[0], s, n_iter=15, use_sparsity=0, use_albedo=0,
                                              lambda_rel=1e-3, diagnostics=True)
    bg = truth[0] == 0
    L = cube[0].astype(np.float64)
    # residual: the fp32 rounding of each plume pixel orthogonal to t (~1e-8 per band) / N
    np.testing.assert_allclose(dg["mu"][15], L[bg].mean(axis=0), rtol=1e-9)


# ---------------------------------------------------------------- P4
def _expected_noiseless(cube, s, truth, use_albedo):
    """Fixed point on the separable scene: alpha_i r_i = LS projection of the plume
    pixel's deviation from the background spectrum onto t = b (.) s (on S)."""
    out = []
    for c in range(cube.shape[0]):
        L = cube[c].astype(np.float64)
        bg = truth[c] == 0
        b = L[bg].mean(axis=0)
        t = b * s.astype(np.float64)
        m = L.mean(axis=0)
        r = L @ m / (m @ m) if use_albedo else np.ones(len(L))
        a = ((L - b) @ t) / (t @ t) / r
        a[bg] = 0.0
        out.append(a)
    return np.array(out)


@pytest.mark.parametrize("use_albedo", [0, 1])
@pytest.mark.parametrize("albedo_scale", [1.0, 0.7])
def test_p4_exact_recovery_without_sparsity(oracle_lib, use_albedo, albedo_scale):
    cube, s, truth = synth.noiseless_scene(cols=2, pixels=400, bands=12, albedo=albedo_scale)
    a, r, st = oracle_lib.retrieve(cube, s, n_iter=14, use_sparsity=0, use_albedo=use_albedo,
                                   lambda_rel=1e-3)
    assert (st == 0).all()
    exp = _expected_noiseless(cube, s, truth, use_albedo)
    plume = truth > 0
    np.testing.assert_allclose(a[plume], exp[plume], rtol=1e-8)
    assert np.abs(a[~plume]).max() < 1e-6
    # and alpha_true recovered to fp32 input rounding
    scale = np.where(use_albedo, 1.0, 1.0)
    np.testing.assert_allclose((a * (r if use_albedo else 1.0))[plume], truth[plume], rtol=2e-6)


def test_p4_recovery_with_sparsity_is_shrunk_by_bias(oracle_lib):
    cube, s, truth = synth.noiseless_scene(cols=2, pixels=400, bands=12)
    a, r, st = oracle_lib.retrieve(cube, s, n_iter=14, use_sparsity=1, use_albedo=1, lambda_rel=1e-3)
    assert (st == 0).all()
    exp = _expected_noiseless(cube, s, truth, 1)
    plume = truth > 0
    assert (a[~plume] == 0).all()                     # background exactly zero
    d = exp[plume] - a[plume]
    assert (d >= -1e-9).all() and d.max() < 0.1       # downward shrinkage w/(r q), tiny here


# ---------------------------------------------------------------- P5
def test_p5_numpy_transcription_10x3(oracle_lib):
    rng = np.random.default_rng(50)
    for _ in range(20):
        L, s = _random_instance(rng, 10, 3, plume_frac=0.3)
        for sp, al in [(1, 1), (0, 1), (1, 0), (0, 0)]:
            for n_iter in (0, 1, 2):
                a, r, rc = oracle_lib.retrieve_column(L, s, n_iter=n_iter, use_sparsity=sp, use_albedo=al,
                                                      lambda_rel=1e-3)
                at, rt = transcription.albedo_rwl1_filter(L, s, n_iter, sp, al, lambda_rel=1e-3)
                assert rc == 0
                np.testing.assert_allclose(a, at, rtol=1e-10, atol=1e-10 * max(1.0, np.abs(at).max()))
                np.testing.assert_allclose(r, rt, rtol=1e-13)


def test_p5_numpy_transcription_tiny_config(oracle_lib):
    cfg = synth.CONFIGS["tiny"]
    cube, s, _ = synth.generate(cfg, columns=[0, 5])
    a, r, st = oracle_lib.retrieve(cube, s, n_iter=cfg.n_iter)
    for j in range(2):
        at, rt = transcription.albedo_rwl1_filter(cube[j], s, cfg.n_iter)
        np.testing.assert_allclose(a[j], at, rtol=1e-8, atol=1e-8 * np.abs(at).max())
        np.testing.assert_allclose(r[j], rt, rtol=1e-13)


# ---------------------------------------------------------------- P6 (sanity, not a pin)
def test_p6_sparsity_sanity_on_generator_scene(oracle_lib):
    cfg = synth.scaled(synth.CONFIGS["segment"], cols=2)
    cube, s, truth = synth.generate(cfg)
    a, r, rc, dg = oracle_lib.retrieve_column(cube[0], s, n_iter=30, diagnostics=True)
    nnz = dg["nnz"]
    assert nnz[30] < nnz[1] < nnz[0]
    tz = truth["alpha"][0] == 0
    zero_frac = (a[tz] == 0).mean()
    assert 0.8 < zero_frac < 1.0
    a0, _, _ = oracle_lib.retrieve_column(cube[0], s, n_iter=0)
    assert (a0 == 0).mean() < 0.01


# ---------------------------------------------------------------- status / edge cases
def test_status_codes_and_nan_fill(oracle_lib):
    rng = np.random.default_rng(60)
    B = 8
    s = -np.full(B, 1e-4, np.float32)
    good = (rng.normal(size=(50, B)) * 0.1 + 3).astype(np.float32)
    few = good[:5]                      # N <= B, rho = 0 -> singular C0
    nonf = good.copy(); nonf[3, 2] = np.nan
    zero = np.zeros_like(good)
    cube = np.stack([good[:5].repeat(10, axis=0) if False else good, nonf, zero])
    a, r, st = oracle_lib.retrieve(cube, s, n_iter=3)
    assert list(st) == [0, 1, 2]
    assert np.isnan(a[1]).all() and np.isnan(a[2]).all() and np.isfinite(a[0]).all()
    a, r, rc = oracle_lib.retrieve_column(few, s, n_iter=3)
    assert rc == 3 and np.isnan(a).all()
    a, r, rc = oracle_lib.retrieve_column(few, s, n_iter=3, lambda_rel=1e-2)
    assert rc == 0
    a, r, rc = oracle_lib.retrieve_column(good, np.zeros(B, np.float32), n_iter=3)
    assert rc == 4
    with pytest.raises(ValueError):
        oracle_lib.retrieve_column(good[:1], s, n_iter=3)


def test_r_floor_reading_c10(oracle_lib):
    """A pixel with r <= r_floor: raw r reported, r~ = r_floor used in the update."""
    rng = np.random.default_rng(61)
    L = (rng.normal(size=(60, 6)) * 0.05 + 2.0).astype(np.float32)
    L[7] = -0.5 * L[8]                  # r_7 < 0
    s = -np.full(6, 1e-4, np.float32)
    a, r, rc = oracle_lib.retrieve_column(L, s, n_iter=0, use_sparsity=0, use_albedo=1)
    a1, r1, rc = oracle_lib.retrieve_column(L, s, n_iter=0, use_sparsity=0, use_albedo=0)
    assert r[7] < 0
    assert a[7] == pytest.approx(a1[7] / 0.05, rel=1e-12)


def test_p6_energy_converges(oracle_lib):
    """P6 sanity (not a pin): the Eq. 8 energy settles -- the paper reports stable
    convergence within 20 iterations; SPEC AC6 asks |E30 - E20| <= 1 %."""
    from paper_2003_02978_b200 import synth
    cfg = synth.CONFIGS["segment"]
    cube, s, _ = synth.generate(cfg, columns=[int(np.flatnonzero(synth.plume_field(cfg).any(axis=1))[0])])
    a, r, rc, dg = oracle_lib.retrieve_column(cube[0], s, n_iter=30, diagnostics=True)
    E = dg["energy"]
    assert rc == 0 and np.isfinite(E).all()
    assert abs(E[30] - E[20]) <= 0.01 * abs(E[30])


# ---------------------------------------------------------------- masking (reading C22)
def test_masked_retrieval_is_retrieval_of_the_valid_rows(oracle_lib):
    """Nodata masking (P:545 censored regions, DESIGN reading C22): a pixel with any band
    non-finite or equal to the nodata value takes no part; the remaining rows are retrieved
    exactly as a column of their own (bitwise), masked pixels read NaN, and a column left
    with < 2 valid rows reports INSUFFICIENT (5) with all-NaN maps."""
    rng = np.random.default_rng(77)
    L, s = _random_instance(rng, 60, 9)
    nodata = np.float32(-9999.0)
    cube = np.stack([L.copy(), L.copy(), L[:3].repeat(20, axis=0)])
    bad = [3, 17, 40]
    cube[0, bad[0], 2] = nodata          # one band equal to nodata
    cube[0, bad[1], 0] = np.nan          # non-finite bands
    cube[0, bad[2], 8] = np.inf
    cube[2, 1:, 4] = nodata              # column 2: one valid row left
    alpha, r, st = oracle_lib.retrieve_masked(cube, s, nodata, n_iter=6)
    keep = np.setdiff1d(np.arange(60), bad)
    a0, r0, rc0 = oracle_lib.retrieve_column(L[keep], s, n_iter=6)
    assert st[0] == rc0 == 0
    assert np.array_equal(alpha[0, keep], a0) and np.array_equal(r[0, keep], r0)
    assert np.all(np.isnan(alpha[0, bad])) and np.all(np.isnan(r[0, bad]))
    a1, r1, _ = oracle_lib.retrieve_column(L, s, n_iter=6)   # nothing masked: plain retrieval
    assert st[1] == 0 and np.array_equal(alpha[1], a1) and np.array_equal(r[1], r1)
    assert st[2] == 5 and np.all(np.isnan(alpha[2])) and np.all(np.isnan(r[2]))
