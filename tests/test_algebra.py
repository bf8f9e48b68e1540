"""The algebra the CUDA path uses in place of the per-iteration covariance (DESIGN.md
5.2 and 5.7), checked on the CPU against the oracle's literal Fig. alg iterates:
  * line 10 summed:   mu^k = mu0 - bbar t'                    (t' = t^{k-1})
  * lines 12-14:      C^k  = C0 + U M U^T,  U = [t', t, h]     (rank-3 identity)
  * Woodbury:         (C^k + rho I)^-1 t = y_t - Y W U^T y_t,  W = M (I + G M)^-1
  * energy trace:     T_k = tr((C^k+rho I)^-1 C0) + bbar^2 t'^T (C^k+rho I)^-1 t'
                            = B - tr(W G) - rho (tr A0^-1 - tr(W Y^T Y)) + bbar^2 (G - G W G)_00
with beta_i = r~_i alpha_i^{k-1}, bbar = mean beta, b2 = mean beta^2, h = mean beta_i (L_i - mu0),
A0 = C0 + rho I, Y = A0^-1 U, G = U^T Y. The oracle recomputes C^k from the residuals."""
import numpy as np
import pytest

from paper_2003_02978_b200 import synth


def _setup(oracle_lib, k, lam=1e-3):
    cfg = synth.scaled(synth.CONFIGS["tiny"], cols=1, pixels=400, bands=10, rank=6)
    cube, s, _ = synth.generate(cfg)
    L = cube[0].astype(np.float64)
    s64 = s.astype(np.float64)
    a, r, rc, dg = oracle_lib.retrieve_column(cube[0], s, n_iter=k, lambda_rel=lam, diagnostics=True)
    assert rc == 0
    rt = np.maximum(r, 0.05)
    alpha_prev = dg["alpha_hist"][k - 1].copy()
    if k - 1 == 0:
        alpha_prev = np.maximum(alpha_prev, 0.0)   # reading C3
    beta = rt * alpha_prev
    mu0, C0 = dg["mu"][0], dg["cov"][0]
    tp = dg["mu"][k - 1] * s64
    return L, s64, dg, beta, mu0, C0, tp, dg["rho"][0]


@pytest.mark.parametrize("k", [1, 2, 5])
def test_rank3_identity_matches_literal_covariance(oracle_lib, k):
    L, s, dg, beta, mu0, C0, tp, rho = _setup(oracle_lib, k)
    N, B = L.shape
    bbar, b2 = beta.mean(), (beta ** 2).mean()
    h = (beta[:, None] * (L - mu0)).mean(axis=0)
    mu = mu0 - bbar * tp
    np.testing.assert_allclose(mu, dg["mu"][k], rtol=1e-13, atol=1e-13 * np.abs(mu).max())
    t = mu * s
    U = np.stack([tp, t, h], axis=1)
    M = np.array([[bbar ** 2, -bbar ** 2, 0.0], [-bbar ** 2, b2, -1.0], [0.0, -1.0, 0.0]])
    Ck = C0 + U @ M @ U.T
    scale = np.sqrt(np.outer(np.diag(dg["cov"][k]), np.diag(dg["cov"][k])))
    assert (np.abs(Ck - dg["cov"][k]) / scale).max() < 1e-12


@pytest.mark.parametrize("k", [1, 3])
def test_woodbury_solve_and_energy_trace(oracle_lib, k):
    L, s, dg, beta, mu0, C0, tp, rho = _setup(oracle_lib, k)
    N, B = L.shape
    bbar, b2 = beta.mean(), (beta ** 2).mean()
    h = (beta[:, None] * (L - mu0)).mean(axis=0)
    t = (mu0 - bbar * tp) * s
    U = np.stack([tp, t, h], axis=1)
    M = np.array([[bbar ** 2, -bbar ** 2, 0.0], [-bbar ** 2, b2, -1.0], [0.0, -1.0, 0.0]])
    A0 = C0 + rho * np.eye(B)
    A0i = np.linalg.inv(A0)
    Y = A0i @ U
    G = U.T @ Y
    W = M @ np.linalg.inv(np.eye(3) + G @ M)
    Ak = dg["cov"][k] + rho * np.eye(B)            # literal C^k from the oracle
    Aki = np.linalg.inv(Ak)
    z = Y[:, 1] - Y @ (W @ (U.T @ Y[:, 1]))
    np.testing.assert_allclose(z, Aki @ t, rtol=1e-8, atol=1e-10 * np.abs(z).max())
    # the z^k the oracle used gives q^k = t.z
    assert abs(t @ z / dg["q"][k] - 1) < 1e-8
    Tk = B - np.trace(W @ G) - rho * (np.trace(A0i) - np.trace(W @ (Y.T @ Y))) + bbar ** 2 * (G - G @ W @ G)[0, 0]
    ref = np.trace(Aki @ C0) + bbar ** 2 * tp @ Aki @ tp
    assert abs(Tk / ref - 1) < 1e-8


def test_energy_from_sufficient_statistics(oracle_lib):
    """E_k = N T_k - 2 sum beta p + q sum beta^2 + sum r~ w alpha, with p_i = (L_i - mu^k).z^k,
    equals the oracle's literal per-pixel Eq. 8 (reading C19)."""
    k = 3
    L, s, dg, beta_prev, mu0, C0, tp, rho = _setup(oracle_lib, k)
    N, B = L.shape
    bbar = beta_prev.mean()
    a, r, rc, _ = oracle_lib.retrieve_column(L.astype(np.float32), s.astype(np.float32), n_iter=k,
                                             lambda_rel=1e-3, diagnostics=True)
    rt = np.maximum(r, 0.05)
    mu, t = dg["mu"][k], dg["mu"][k] * s
    Ak = dg["cov"][k] + rho * np.eye(B)
    Aki = np.linalg.inv(Ak)
    z = Aki @ t
    q = t @ z
    alpha = dg["alpha_hist"][k]
    beta = rt * alpha
    p = (L - mu) @ z
    w = 1.0 / (dg["alpha_hist"][k - 1] + 1e-2)
    Tk = np.trace(Aki @ C0) + bbar ** 2 * tp @ Aki @ tp
    E = N * Tk - 2 * np.sum(beta * p) + q * np.sum(beta ** 2) + np.sum(rt * w * alpha)
    assert abs(E / dg["energy"][k] - 1) < 1e-9
