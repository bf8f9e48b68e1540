"""Pins for the oracle's step functions (CPU only).

Each step is checked against hand-worked examples (tests/golden/spec_examples.json,
cited per entry) and against textbook library routines (math.fsum, numpy.cov,
numpy.linalg.cholesky, scipy.linalg.cho_solve, scipy.optimize), never against a
retyped copy of its own formula.
"""
import json
import math
import os

import numpy as np
import pytest
import scipy.linalg
import scipy.optimize

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def test_mean_examples(oracle_lib):
    for ex in GOLD["mean"]:
        np.testing.assert_array_equal(oracle_lib.mean(np.array(ex["L"], float)), ex["expected"], ex["cite"])


def test_mean_matches_exactly_rounded_sum(oracle_lib):
    rng = np.random.default_rng(0)
    L = rng.normal(3.0, 2.0, size=(100, 7))
    mu = oracle_lib.mean(L)
    ref = np.array([math.fsum(L[:, b]) / 100 for b in range(7)])
    np.testing.assert_allclose(mu, ref, rtol=1e-13, atol=0)


def test_covariance_examples(oracle_lib):
    for ex in GOLD["covariance"]:
        np.testing.assert_allclose(oracle_lib.covariance(np.array(ex["L"], float)), ex["expected"],
                                   atol=1e-15, err_msg=ex["cite"])


def test_covariance_matches_numpy_population_cov(oracle_lib):
    rng = np.random.default_rng(1)
    L = rng.normal(size=(50, 6)) @ rng.normal(size=(6, 6)) + 5.0
    C = oracle_lib.covariance(L)
    np.testing.assert_allclose(C, np.cov(L, rowvar=False, bias=True), rtol=1e-10, atol=1e-12)
    assert np.array_equal(C, C.T)
    assert np.linalg.eigvalsh(C).min() >= -1e-10 * np.trace(C)


def test_cholesky_matches_numpy_and_detects_non_spd(oracle_lib):
    rng = np.random.default_rng(2)
    X = rng.normal(size=(9, 9))
    A = X @ X.T + 0.5 * np.eye(9)
    G, rc = oracle_lib.cholesky(A)
    assert rc == 0
    np.testing.assert_allclose(np.tril(G), np.linalg.cholesky(A), rtol=1e-12, atol=1e-13)
    _, rc = oracle_lib.cholesky(np.array([[1.0, 2.0], [2.0, 1.0]]))
    assert rc == 2          # second pivot 1 - 4 < 0
    _, rc = oracle_lib.cholesky(np.array([[0.0, 0.0], [0.0, 1.0]]))
    assert rc == 1


def test_spd_solve_examples_and_residual(oracle_lib):
    for ex in GOLD["spd_solve"]:
        np.testing.assert_allclose(oracle_lib.spd_solve(np.array(ex["A"], float), np.array(ex["b"], float)),
                                   ex["expected"], rtol=1e-15, err_msg=ex["cite"])
    rng = np.random.default_rng(3)
    X = rng.normal(size=(6, 6))
    A = X @ X.T + np.eye(6)
    v = rng.normal(size=6)
    x = oracle_lib.spd_solve(A, v)
    assert np.linalg.norm(A @ x - v) <= 1e-10 * np.linalg.norm(v)
    np.testing.assert_allclose(x, scipy.linalg.cho_solve(scipy.linalg.cho_factor(A), v), rtol=1e-11)
    # ridge: (A + rho I)^-1 v
    x2 = oracle_lib.spd_solve(A, v, rho=0.25)
    np.testing.assert_allclose(x2, np.linalg.solve(A + 0.25 * np.eye(6), v), rtol=1e-11)
    with pytest.raises(np.linalg.LinAlgError):
        oracle_lib.spd_solve(np.zeros((3, 3)), v[:3])


def test_albedo_examples(oracle_lib):
    for ex in GOLD["albedo"]:
        assert oracle_lib.albedo(np.array(ex["L"], float), np.array(ex["mu"], float)) == pytest.approx(
            ex["expected"], abs=1e-15), ex["cite"]


def test_reweight_examples(oracle_lib):
    for ex in GOLD["reweight"]:
        assert oracle_lib.reweight(ex["alpha"], ex["eps"]) == pytest.approx(ex["expected"], rel=1e-14), ex["cite"]


def test_ista_update_examples_and_signed_zero(oracle_lib):
    for ex in GOLD["ista_update"]:
        assert oracle_lib.ista_update(ex["num"], ex["w"], ex["r"], ex["q"]) == pytest.approx(
            ex["expected"], rel=1e-14, abs=0), ex["cite"]
    # reading C14: max(x, 0) is canonical +0, also for x = -0 and for x < 0
    for num, w in [(0.0, 0.0), (-0.0, 0.0), (1.0, 1.0), (-3.0, 0.0)]:
        v = oracle_lib.ista_update(num, w, 1.0, 2.0)
        assert v == 0.0 and math.copysign(1.0, v) == 1.0


def test_ista_update_is_exact_prox_minimiser(oracle_lib):
    """Eq. 6 / line 16 is the exact minimiser of J(a) = 1/2 q r^2 a^2 - r num a + r w a
    over a >= 0 (the per-pixel objective of reading C4); checked by bounded
    scalar minimisation (scipy) on random instances (SPEC AC8 analogue)."""
    rng = np.random.default_rng(4)
    for _ in range(200):
        num, w = rng.normal() * 3, abs(rng.normal()) * 2
        r, q = rng.uniform(0.2, 2.0), rng.uniform(0.1, 3.0)
        J = lambda a: 0.5 * q * r * r * a * a - r * num * a + r * w * a
        hi = max(10.0, 4 * abs(num) / (q * r))
        res = scipy.optimize.minimize_scalar(J, bounds=(0.0, hi), method="bounded",
                                             options={"xatol": 1e-12})
        a_bf = res.x if J(res.x) < J(0.0) else 0.0
        assert oracle_lib.ista_update(num, w, r, q) == pytest.approx(a_bf, abs=1e-6)


def test_closed_form_examples(oracle_lib):
    for ex in GOLD["closed_form"]:
        a = oracle_lib.mf_closed_form(np.array(ex["L"], float), np.array(ex["mu"], float),
                                      np.array(ex["C"], float), np.array(ex["t"], float))
        np.testing.assert_allclose(a, ex["expected"], rtol=1e-14, atol=1e-15, err_msg=ex["cite"])


def test_closed_form_is_gls_estimate(oracle_lib):
    """Eq. 3 is the generalised-least-squares estimate of a in L - mu = a t + n,
    n ~ N(0, C): compare with whitened least squares via scipy.linalg.lstsq."""
    rng = np.random.default_rng(5)
    B, N = 6, 20
    X = rng.normal(size=(B, B))
    C = X @ X.T + 0.3 * np.eye(B)
    mu, t = rng.normal(size=B), rng.normal(size=B)
    L = mu + rng.normal(size=(N, B))
    a = oracle_lib.mf_closed_form(L, mu, C, t)
    W = np.linalg.inv(np.linalg.cholesky(C))       # whitening: W C W^T = I
    for i in range(N):
        sol, *_ = scipy.linalg.lstsq((W @ t)[:, None], W @ (L[i] - mu))
        assert a[i] == pytest.approx(sol[0], rel=1e-10, abs=1e-12)


# ---- energy, Eq. 8, the objective of Fig. 4 ----------------
def test_energy_closed_form_NB(oracle_lib):
    """alpha = 0, w = 0 with mu, C the sample mean / population covariance: the
    quadratic term is sum_i (L_i-mu)^T C^-1 (L_i-mu) = N tr(C^-1 C) = N B exactly."""
    rng = np.random.default_rng(11)
    N, B = 40, 5
    L = rng.normal(size=(N, B)) @ rng.normal(size=(B, B)) + 3.0
    mu = L.mean(axis=0)
    C = (L - mu).T @ (L - mu) / N
    E = oracle_lib.energy(L, mu, C, np.ones(B), np.zeros(N), np.ones(N))
    assert abs(E - N * B) < 1e-9 * N * B


def test_energy_exact_fit_and_penalty(oracle_lib):
    """L_i = mu + r~_i alpha_i t makes every residual d_i zero: E is then
    the penalty sum_i r~_i w_i |alpha_i| alone."""
    rng = np.random.default_rng(12)
    N, B = 12, 4
    mu, t = rng.uniform(1, 2, B), -rng.uniform(0.1, 0.2, B)
    alpha, rt, w = rng.uniform(0, 5, N), rng.uniform(0.5, 1.5, N), rng.uniform(0, 2, N)
    L = mu + (rt * alpha)[:, None] * t
    A = rng.normal(size=(B, B))
    C = A @ A.T + B * np.eye(B)
    assert abs(oracle_lib.energy(L, mu, C, t, alpha, rt)) < 1e-20
    E = oracle_lib.energy(L, mu, C, t, alpha, rt, w)
    assert abs(E - np.sum(rt * w * alpha)) < 1e-12 * np.sum(rt * w * alpha)


def test_energy_matches_direct_sum(oracle_lib):
    """Random 10-pixel instance vs the term-by-term sum with numpy's inverse."""
    rng = np.random.default_rng(13)
    N, B = 10, 3
    L, mu, t = rng.normal(size=(N, B)), rng.normal(size=B), rng.normal(size=B)
    alpha, rt, w = rng.uniform(-1, 3, N), rng.uniform(0.5, 1.5, N), rng.uniform(0, 1, N)
    A = rng.normal(size=(B, B))
    C, rho = A @ A.T + 0.1 * np.eye(B), 0.3
    Ci = np.linalg.inv(C + rho * np.eye(B))
    d = L - (rt * alpha)[:, None] * t - mu
    ref = np.einsum("ib,bc,ic->", d, Ci, d) + np.sum(rt * w * np.abs(alpha))
    assert abs(oracle_lib.energy(L, mu, C, t, alpha, rt, w, rho) - ref) < 1e-10 * abs(ref)


def test_energy_trace_wiring(oracle_lib):
    """The retrieval's energy trace E_k (reading C19) equals Eq. 8 evaluated with the
    iteration's own mu^k, C^k (+ rho), t^k = mu^k (.) s, w^k = 1/(alpha^{k-1} + eps) and
    the updated alpha^k (alpha^0 clamped when N_iter >= 1, w^0 = 0)."""
    from paper_2003_02978_b200 import synth
    cfg = synth.scaled(synth.CONFIGS["tiny"], cols=1, pixels=300, bands=8, rank=4)
    cube, s, _ = synth.generate(cfg)
    L = cube[0].astype(np.float64)
    eps, lam, K = 1e-2, 1e-3, 4
    a, r, rc, dg = oracle_lib.retrieve_column(cube[0], s, n_iter=K, eps=eps, lambda_rel=lam,
                                              diagnostics=True)
    assert rc == 0
    rt = np.maximum(r, 0.05)
    rho = dg["rho"][0]
    prev = None
    for k in range(K + 1):
        alpha = dg["alpha_hist"][k]
        if k == 0:
            alpha = np.maximum(alpha, 0.0)
        t = dg["mu"][k] * s.astype(np.float64)
        w = None if k == 0 else 1.0 / (prev + eps)
        E = oracle_lib.energy(L, dg["mu"][k], dg["cov"][k], t, alpha, rt, w, rho)
        assert abs(E - dg["energy"][k]) <= 1e-12 * abs(E)
        prev = alpha
