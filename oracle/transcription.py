"""Second, independent transcription of AlbedoReWeightL1Filter (PAPER.md Fig. alg,
P:295-393) in numpy fp64, for tiny inputs.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). Written line by line from the
figure, independently of smf_oracle.c (matrix algebra via numpy instead of loops;
linear solves via numpy.linalg.solve instead of a hand Cholesky). Same readings
C1, C3, C8, C9, C10, C14.
"""
from __future__ import annotations

import numpy as np


def albedo_rwl1_filter(D, s, n_iter, use_sparsity=True, use_albedo=True, eps=1e-2,
                       lambda_rel=0.0, r_floor=0.05):
    """D: [N][B] radiance of one partition. Returns (alpha, r)."""
    L = np.asarray(D, dtype=np.float32).astype(np.float64)
    s = np.asarray(s, dtype=np.float32).astype(np.float64)
    N, B = L.shape
    # line 2
    mu0 = L.sum(axis=0) / N
    # line 3 (outer products)
    Y = L - mu0
    C0 = (Y.T @ Y) / N
    rho = lambda_rel * np.trace(C0) / B
    I = np.eye(B)
    # lines 4-5
    if use_albedo:
        r = (L @ mu0) / (mu0 @ mu0)
        rt = np.maximum(r, r_floor)
    else:
        r = np.ones(N)
        rt = np.ones(N)
    # line 6
    t0 = mu0 * s
    Cit = np.linalg.solve(C0 + rho * I, t0)
    alpha = (Y @ Cit) / (rt * (t0 @ Cit))
    if n_iter == 0:
        return alpha, r
    alpha = np.where(alpha > 0, alpha, 0.0)
    mu_prev = mu0
    for _k in range(1, n_iter + 1):
        # line 9
        w = 1.0 / (alpha + eps) if use_sparsity else np.zeros(N)
        # line 10
        mu = (L - (rt * alpha)[:, None] * (mu_prev * s)[None, :]).sum(axis=0) / N
        # lines 11-13
        t = mu * s
        d = L - (rt * alpha)[:, None] * t[None, :] - mu[None, :]
        # line 14
        C = (d.T @ d) / N
        # line 16
        Cit = np.linalg.solve(C + rho * I, t)
        x = ((L - mu) @ Cit - w) / (rt * (t @ Cit))
        alpha = np.where(x > 0, x, 0.0)
        mu_prev = mu
    return alpha, r
