"""fp64 CPU oracle for the albedo-corrected reweighted-l1 matched filter.

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package. The product
path (paper_2003_02978_b200) never imports it and shares no code with it.

`smf_oracle.c` is the literal Fig. alg transcription in
fp64 C with OpenMP over columns; `transcription.py` is an independent numpy
transcription used to cross-check it on tiny inputs.

Parity status per function:
  oracle_mean, oracle_second_moment, oracle_cholesky/spd_solve, oracle_albedo,
  oracle_reweight, oracle_ista_update, oracle_mf_closed_form -- pinned by the
  paper's/SPEC's worked examples and textbook routines (tests/test_oracle_steps.py).
  oracle_retrieve(_column) -- pinned by brute-force minimisation (P1), the
  closed-form MF (P2), invariants (P3), exact recovery on a noiseless scene (P4)
  and the numpy transcription (P5) (tests/test_oracle_pins.py). Its absolute
  maps on noisy scenes beyond those pins are "parity unpinned".
  oracle_energy / the energy trace (Eq. 8, reading C19) -- pinned by E = N*B at
  alpha = 0, E = penalty at an exact fit, a direct per-pixel sum and the trace
  wiring (tests/test_oracle_steps.py).
  retrieve_masked (reading C22) -- the valid rows retrieved as a column of their own,
  pinned bitwise against retrieve_column on the filtered rows, NaN fill and the
  INSUFFICIENT status (tests/test_oracle_pins.py).
  Detector grouping (reading C20) has no function of its own: a partition of G
  columns is retrieve_column on their pooled pixels (pixel-permutation invariance,
  P3, pins the pooling order).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "smf_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

STATUS = {0: "OK", 1: "NONFINITE", 2: "DEGENERATE_MEAN", 3: "NOT_SPD", 4: "DEGENERATE_TARGET",
          5: "BAD_ARG", 6: "NOMEM"}

_d = ctypes.POINTER(ctypes.c_double)
_f = ctypes.POINTER(ctypes.c_float)
_i32 = ctypes.POINTER(ctypes.c_int32)
_i64 = ctypes.POINTER(ctypes.c_int64)


class _Diag(ctypes.Structure):
    _fields_ = [("mu", _d), ("cov", _d), ("q", _d), ("alpha_hist", _d), ("nnz", _i64), ("rho", _d),
                ("energy", _d)]


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (-O2, OpenMP). Building the checker is not using it."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        L = _lib
        L.oracle_mean.argtypes = [ctypes.c_int, ctypes.c_int, _d, _d]
        L.oracle_second_moment.argtypes = [ctypes.c_int, ctypes.c_int, _d, _d]
        L.oracle_cholesky.argtypes = [ctypes.c_int, _d]
        L.oracle_cholesky.restype = ctypes.c_int
        L.oracle_chol_solve.argtypes = [ctypes.c_int, _d, _d, _d]
        L.oracle_spd_solve.argtypes = [ctypes.c_int, _d, ctypes.c_double, _d, _d]
        L.oracle_spd_solve.restype = ctypes.c_int
        L.oracle_albedo.argtypes = [ctypes.c_int, _d, _d]
        L.oracle_albedo.restype = ctypes.c_double
        L.oracle_reweight.argtypes = [ctypes.c_double, ctypes.c_double]
        L.oracle_reweight.restype = ctypes.c_double
        L.oracle_ista_update.argtypes = [ctypes.c_double] * 4
        L.oracle_ista_update.restype = ctypes.c_double
        L.oracle_mf_closed_form.argtypes = [ctypes.c_int, ctypes.c_int, _d, _d, _d, _d, _d]
        L.oracle_mf_closed_form.restype = ctypes.c_int
        L.oracle_retrieve_column.argtypes = [_f, ctypes.c_int, ctypes.c_int, _f, ctypes.c_int,
                                             ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                             ctypes.c_double, ctypes.c_double, _d, _d,
                                             ctypes.POINTER(_Diag)]
        L.oracle_retrieve_column.restype = ctypes.c_int
        L.oracle_retrieve.argtypes = [_f, ctypes.c_int, ctypes.c_int, ctypes.c_int, _f, ctypes.c_int,
                                      ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                      ctypes.c_double, _d, _d, _i32, ctypes.c_int]
        L.oracle_retrieve.restype = ctypes.c_int
        L.oracle_max_threads.restype = ctypes.c_int
        L.oracle_energy.argtypes = [ctypes.c_int, ctypes.c_int, _d, _d, _d, ctypes.c_double, _d, _d, _d, _d]
        L.oracle_energy.restype = ctypes.c_double
    return _lib


def _p(a, t):
    return a.ctypes.data_as(t)


def _c64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ---- step functions ---------------------------------------------------------

def mean(L):
    L = _c64(L)
    mu = np.empty(L.shape[1])
    lib().oracle_mean(L.shape[0], L.shape[1], _p(L, _d), _p(mu, _d))
    return mu


def second_moment(D):
    D = _c64(D)
    C = np.empty((D.shape[1], D.shape[1]))
    lib().oracle_second_moment(D.shape[0], D.shape[1], _p(D, _d), _p(C, _d))
    return C


def covariance(L):
    """Fig. alg line 3: (1/N) sum (L_i - mu0)(L_i - mu0)^T."""
    L = _c64(L)
    return second_moment(L - mean(L)[None, :])


def cholesky(A):
    G = _c64(A).copy()
    rc = lib().oracle_cholesky(G.shape[0], _p(G, _d))
    return G, rc


def spd_solve(A, b, rho=0.0):
    A, b = _c64(A), _c64(b)
    x = np.empty_like(b)
    rc = lib().oracle_spd_solve(A.shape[0], _p(A, _d), float(rho), _p(b, _d), _p(x, _d))
    if rc:
        raise np.linalg.LinAlgError(STATUS[rc])
    return x


def albedo(L, mu):
    L, mu = _c64(L), _c64(mu)
    return lib().oracle_albedo(L.shape[0], _p(L, _d), _p(mu, _d))


def reweight(alpha_prev, eps):
    return lib().oracle_reweight(float(alpha_prev), float(eps))


def ista_update(num, w, r, q):
    return lib().oracle_ista_update(float(num), float(w), float(r), float(q))


def mf_closed_form(L, mu, C, t):
    L, mu, C, t = _c64(L), _c64(mu), _c64(C), _c64(t)
    a = np.empty(L.shape[0])
    rc = lib().oracle_mf_closed_form(L.shape[0], L.shape[1], _p(L, _d), _p(mu, _d), _p(C, _d),
                                     _p(t, _d), _p(a, _d))
    if rc:
        raise np.linalg.LinAlgError(STATUS[rc])
    return a


# ---- the procedure ------------------------------------------------------------

DEFAULTS = dict(n_iter=30, use_sparsity=True, use_albedo=True, eps=1e-2, lambda_rel=0.0,
                r_floor=0.05)


def energy(L, mu, C, t, alpha, rt, w=None, rho=0.0):
    """Eq. 8 as printed: sum_i d_i^T (C+rho I)^-1 d_i + r~_i w_i |alpha_i|,
    d_i = L_i - r~_i alpha_i t - mu (fp64; NaN if C + rho I is not SPD)."""
    L, mu, C, t, alpha, rt = map(_c64, (L, mu, C, t, alpha, rt))
    N, B = L.shape
    wp = _p(_c64(w), _d) if w is not None else None
    return lib().oracle_energy(N, B, _p(L, _d), _p(mu, _d), _p(C, _d), float(rho), _p(t, _d),
                               _p(alpha, _d), _p(rt, _d), wp)


def retrieve_column(L, s, n_iter=30, use_sparsity=True, use_albedo=True, eps=1e-2,
                    lambda_rel=0.0, r_floor=0.05, diagnostics=False):
    """One partition. L fp32 [N][B]. Returns (alpha, r, status[, diag dict])."""
    L = np.ascontiguousarray(L, dtype=np.float32)
    s = np.ascontiguousarray(s, dtype=np.float32)
    N, B = L.shape
    alpha = np.empty(N)
    r = np.empty(N)
    dg = None
    out = {}
    if diagnostics:
        K = n_iter + 1
        out = dict(mu=np.zeros((K, B)), cov=np.zeros((K, B, B)), q=np.zeros(K),
                   alpha_hist=np.zeros((K, N)), nnz=np.zeros(K, dtype=np.int64), rho=np.zeros(1),
                   energy=np.zeros(K))
        dg = _Diag(_p(out["mu"], _d), _p(out["cov"], _d), _p(out["q"], _d),
                   _p(out["alpha_hist"], _d), _p(out["nnz"], _i64), _p(out["rho"], _d),
                   _p(out["energy"], _d))
    rc = lib().oracle_retrieve_column(_p(L, _f), N, B, _p(s, _f), int(n_iter), int(use_sparsity),
                                      int(use_albedo), float(eps), float(lambda_rel),
                                      float(r_floor), _p(alpha, _d), _p(r, _d),
                                      ctypes.byref(dg) if dg is not None else None)
    if rc == 5:
        raise ValueError("invalid argument")
    if diagnostics:
        return alpha, r, rc, out
    return alpha, r, rc


def retrieve_masked(cube, s, nodata, **kw):
    """Nodata masking (the paper skips censored regions): per column, a pixel with
    any band non-finite or equal to `nodata` is removed before Fig. alg runs on the
    remaining rows (so every statistic uses only valid pixels, N = their count); its
    alpha and r are NaN. Fewer than 2 valid pixels: status 5 (INSUFFICIENT), all NaN.
    Returns (alpha, r, status[, energies [n_iter+1][cols] if diagnostics=True])."""
    cube = np.asarray(cube, dtype=np.float32)
    cols, N, B = cube.shape
    diagnostics = kw.pop("diagnostics", False)
    alpha = np.full((cols, N), np.nan)
    r = np.full((cols, N), np.nan)
    status = np.zeros(cols, dtype=np.int32)
    energy = np.full((kw.get("n_iter", 30) + 1, cols), np.nan)
    for c in range(cols):
        ok = np.all(np.isfinite(cube[c]) & (cube[c] != np.float32(nodata)), axis=1)
        if ok.sum() < 2:
            status[c] = 5
            continue
        out = retrieve_column(cube[c][ok], s, diagnostics=diagnostics, **kw)
        a, rr, rc = out[:3]
        alpha[c, ok], r[c, ok], status[c] = a, rr, rc
        if rc != 0:
            alpha[c], r[c] = np.nan, np.nan
        if diagnostics:
            energy[:, c] = out[3]["energy"]
    if diagnostics:
        return alpha, r, status, energy
    return alpha, r, status


def retrieve(cube, s, n_iter=30, use_sparsity=True, use_albedo=True, eps=1e-2, lambda_rel=0.0,
             r_floor=0.05, threads=0):
    """Whole cube fp32 [cols][N][B] -> (alpha fp64 [cols][N], r fp64 [cols][N], status int32 [cols])."""
    cube = np.ascontiguousarray(cube, dtype=np.float32)
    s = np.ascontiguousarray(s, dtype=np.float32)
    cols, N, B = cube.shape
    alpha = np.empty((cols, N))
    r = np.empty((cols, N))
    status = np.empty(cols, dtype=np.int32)
    if N < 2 or B < 1:
        raise ValueError("invalid argument")
    lib().oracle_retrieve(_p(cube, _f), cols, N, B, _p(s, _f), int(n_iter), int(use_sparsity),
                          int(use_albedo), float(eps), float(lambda_rel), float(r_floor),
                          _p(alpha, _d), _p(r, _d), _p(status, _i32), int(threads))
    return alpha, r, status


def max_threads() -> int:
    return lib().oracle_max_threads()
