"""Seeded synthetic AVIRIS-NG-shaped radiance scenes (shared input generator).

This module is the ONLY code shared by the CUDA path's tests/bench and the CPU
oracle's tests. It holds none of the retrieval method's arithmetic: it draws
background spectra, correlated noise, albedo fields and plume fields, and
applies the forward model x * (1 - k * alpha) that BASELINE.json's configs
name (the linearised Beer-Lambert model, Eq. 1; sign
convention s = dlnL/d(ppm m) <= 0).

The real inputs of the paper (AVIRIS-NG flightlines ang20160211t075004 and
ang20160214t051014, MODTRAN6 unit absorption spectra, LES plumes; P:475,
P:493) are not available; these seeded scenes stand in for
them with the shapes of BASELINE.json's configs (recipe
restated in DESIGN.md section 3).

Layout of every cube: float32, C-contiguous [cols][pixels][bands]
(detector column major; pixels are along-track lines).

Determinism: every random component of column c is drawn from
``SeedSequence(seed, spawn_key=(component, c))`` so a column's data does not
depend on which other columns are generated (the oracle can regenerate a
sampled column alone). Scene-level fields (albedo field, plume field) are
drawn once per scene from their own spawn keys and sliced.
"""
from __future__ import annotations

import dataclasses
import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

GENERATOR_VERSION = 3

# spawn-key components
_K_ABSORB, _K_SPECTRUM, _K_NOISE, _K_ALBEDO, _K_PLUME = 1, 2, 3, 4, 5


@dataclasses.dataclass(frozen=True)
class SceneConfig:
    name: str
    cols: int
    pixels: int
    bands: int
    n_iter: int
    rank: int
    wl_lo: float
    wl_hi: float
    absorb_lo: float          # absorbing window for the unit absorption spectrum
    absorb_hi: float
    albedo: tuple             # ("iid", lo, hi) | ("smooth", lo, hi, sigma_px)
    plume: tuple              # ("sparse", frac, lo, hi) | ("ellipses", coverages, peak_lo, peak_hi)
    seed: int
    use_sparsity: bool = True
    use_albedo: bool = True

    @property
    def n_pix(self) -> int:
        return self.cols * self.pixels

    @property
    def cube_bytes(self) -> int:
        return self.cols * self.pixels * self.bands * 4


def _cfg(**kw) -> SceneConfig:
    return SceneConfig(**kw)


# BASELINE.json "configs" (index in comments). Constants BASELINE.json does not
# fix are the SURVEY.md 8(d) proposals, marked (p) there and in DESIGN.md.
CONFIGS = {
    # configs[0]
    "tiny": _cfg(name="tiny", cols=8, pixels=512, bands=32, n_iter=10, rank=8,
                 wl_lo=2122.0, wl_hi=2488.0, absorb_lo=2122.0, absorb_hi=2488.0,
                 albedo=("iid", 0.5, 1.5), plume=("sparse", 0.02, 500.0, 3000.0), seed=1),
    # configs[1]
    "segment": _cfg(name="segment", cols=598, pixels=2000, bands=72, n_iter=30, rank=16,
                    wl_lo=2122.0, wl_hi=2488.0, absorb_lo=2122.0, absorb_hi=2488.0,
                    albedo=("iid", 0.5, 1.5), plume=("ellipses", (0.005,), 4000.0, 4000.0), seed=2),
    # configs[2] -- the headline throughput case
    "flightline": _cfg(name="flightline", cols=598, pixels=20000, bands=72, n_iter=30, rank=16,
                       wl_lo=2122.0, wl_hi=2488.0, absorb_lo=2122.0, absorb_hi=2488.0,
                       albedo=("smooth", 0.3, 1.7, 8.0),
                       plume=("ellipses", (0.001, 0.003, 0.005, 0.007, 0.01), 2000.0, 8000.0), seed=3),
    # configs[3]
    "stress": _cfg(name="stress", cols=598, pixels=4000, bands=425, n_iter=30, rank=32,
                   wl_lo=380.0, wl_hi=2510.0, absorb_lo=2100.0, absorb_hi=2500.0,
                   albedo=("iid", 0.5, 1.5), plume=("ellipses", (0.005,), 4000.0, 4000.0), seed=4),
}
# configs[4]: campaign of 4 flightlines, plume densities 0 / 0.1 / 1 / 5 %
for _j, (_frac, _seed) in enumerate(zip((0.0, 0.001, 0.01, 0.05), (10, 11, 12, 13))):
    CONFIGS[f"campaign{_j}"] = _cfg(
        name=f"campaign{_j}", cols=598, pixels=12000, bands=72, n_iter=30, rank=16,
        wl_lo=2122.0, wl_hi=2488.0, absorb_lo=2122.0, absorb_hi=2488.0,
        albedo=("iid", 0.5, 1.5), plume=("sparse", _frac, 500.0, 3000.0), seed=_seed)


def scaled(cfg: SceneConfig, **changes) -> SceneConfig:
    """Same generator recipe, different shape (e.g. fewer columns for tests)."""
    return dataclasses.replace(cfg, **changes)


def _rng(seed: int, *key: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(seed, spawn_key=tuple(key))))


def wavelengths(cfg: SceneConfig) -> np.ndarray:
    return np.linspace(cfg.wl_lo, cfg.wl_hi, cfg.bands)


def absorption_k(cfg: SceneConfig) -> np.ndarray:
    """k(lambda) >= 0: 4 Gaussian absorption lines (BASELINE.json configs[0]).

    s = -k is the unit absorption spectrum handed to the retrieval.
    """
    rng = _rng(cfg.seed, _K_ABSORB)
    wl = wavelengths(cfg)
    dwl = (cfg.wl_hi - cfg.wl_lo) / max(cfg.bands - 1, 1)
    span = cfg.absorb_hi - cfg.absorb_lo
    k = np.zeros(cfg.bands)
    for _ in range(4):
        d = rng.uniform(0.3, 1.0) * 5e-5
        c = rng.uniform(cfg.absorb_lo + 0.1 * span, cfg.absorb_hi - 0.1 * span)
        w = rng.uniform(1.0, 3.0) * dwl
        k += d * np.exp(-0.5 * ((wl - c) / w) ** 2)
    k[(wl < cfg.absorb_lo) | (wl > cfg.absorb_hi)] = 0.0
    return k


def unit_absorption(cfg: SceneConfig) -> np.ndarray:
    """s = dlnL/d(ppm m) as float32 (negative in absorption bands)."""
    return (-absorption_k(cfg)).astype(np.float32)


def _column_spectrum(cfg: SceneConfig, c: int):
    rng = _rng(cfg.seed, _K_SPECTRUM, c)
    wl = wavelengths(cfg)
    span = cfg.wl_hi - cfg.wl_lo
    b = np.ones(cfg.bands)
    for _ in range(3):
        a = rng.uniform(1.0, 3.0)
        cc = rng.uniform(cfg.wl_lo, cfg.wl_hi)
        w = rng.uniform(0.15, 0.5) * span
        b += a * np.exp(-0.5 * ((wl - cc) / w) ** 2)
    g = rng.standard_normal((cfg.bands, cfg.rank))
    F = (0.05 * b)[:, None] * g / math.sqrt(cfg.rank)
    return b, F


def albedo_field(cfg: SceneConfig) -> np.ndarray:
    """Per-pixel albedo a[cols][pixels] (float64)."""
    rng = _rng(cfg.seed, _K_ALBEDO)
    kind = cfg.albedo[0]
    if kind == "iid":
        _, lo, hi = cfg.albedo
        return rng.uniform(lo, hi, size=(cfg.cols, cfg.pixels))
    if kind == "smooth":
        from scipy.ndimage import gaussian_filter
        from scipy.special import ndtr
        _, lo, hi, sigma = cfg.albedo
        wn = rng.standard_normal((cfg.cols, cfg.pixels)).astype(np.float32)
        f = gaussian_filter(wn, sigma=sigma, mode="wrap").astype(np.float64)
        f = (f - f.mean()) / f.std()
        return lo + (hi - lo) * ndtr(f)
    raise ValueError(kind)


def _ellipse(alpha: np.ndarray, rng: np.random.Generator, coverage: float, peak: float) -> None:
    """Add one elliptical Gaussian plume alpha = peak*exp(-Q/2) (3:1 axes, random
    orientation, centre in the middle 50% of the image), zero below 100 ppm m,
    with its sigma bisected so the support is `coverage` of the pixels."""
    cols, n = alpha.shape
    cx = rng.uniform(0.25, 0.75) * cols
    cy = rng.uniform(0.25, 0.75) * n
    th = rng.uniform(0.0, math.pi)
    target = coverage * cols * n
    cut = 2.0 * math.log(peak / 100.0)

    def field(sig):
        half = int(3.0 * sig * math.sqrt(cut)) + 2
        x0, x1 = max(0, int(cx) - half), min(cols, int(cx) + half + 1)
        y0, y1 = max(0, int(cy) - half), min(n, int(cy) + half + 1)
        X, Y = np.meshgrid(np.arange(x0, x1) + 0.5 - cx, np.arange(y0, y1) + 0.5 - cy, indexing="ij")
        u = math.cos(th) * X + math.sin(th) * Y
        v = -math.sin(th) * X + math.cos(th) * Y
        Q = (u / (3.0 * sig)) ** 2 + (v / sig) ** 2
        a = peak * np.exp(-0.5 * Q)
        a[a < 100.0] = 0.0
        return (x0, x1, y0, y1), a

    lo, hi = 0.1, 10.0
    while field(hi)[1].astype(bool).sum() < target:
        hi *= 2.0
    for _ in range(60):
        mid = 0.5 * (lo + hi)
        if np.count_nonzero(field(mid)[1]) < target:
            lo = mid
        else:
            hi = mid
    (x0, x1, y0, y1), a = field(hi)
    alpha[x0:x1, y0:y1] += a


def plume_field(cfg: SceneConfig) -> np.ndarray:
    """True enhancement alpha[cols][pixels] in ppm m (float64)."""
    rng = _rng(cfg.seed, _K_PLUME)
    alpha = np.zeros((cfg.cols, cfg.pixels))
    kind = cfg.plume[0]
    if kind == "sparse":
        _, frac, lo, hi = cfg.plume
        npix = cfg.cols * cfg.pixels
        m = int(math.ceil(frac * npix))
        if m:
            idx = rng.choice(npix, size=m, replace=False)
            alpha.reshape(-1)[idx] = rng.uniform(lo, hi, size=m)
    elif kind == "ellipses":
        _, coverages, plo, phi = cfg.plume
        for cov in coverages:
            peak = plo if plo == phi else rng.uniform(plo, phi)
            _ellipse(alpha, rng, cov, peak)
    else:
        raise ValueError(kind)
    return alpha


def _fill_column(cfg, c, k, albedo, alpha, out):
    b, F = _column_spectrum(cfg, c)
    rng = _rng(cfg.seed, _K_NOISE, c)
    g = rng.standard_normal((cfg.pixels, cfg.rank), dtype=np.float32)
    e = rng.standard_normal((cfg.pixels, cfg.bands), dtype=np.float32)
    x = albedo[:, None] * b[None, :] + g.astype(np.float64) @ F.T + (0.01 * b)[None, :] * e
    x *= 1.0 - k[None, :] * alpha[:, None]
    out[...] = x.astype(np.float32)


def generate(cfg: SceneConfig, columns=None, threads: int | None = None):
    """Return (radiance float32 [len(columns)][pixels][bands], s float32 [bands],
    truth dict with 'alpha' and 'albedo' (float64 [cols][pixels]))."""
    cols = list(range(cfg.cols)) if columns is None else [int(c) for c in columns]
    k = absorption_k(cfg)
    albedo = albedo_field(cfg)
    alpha = plume_field(cfg)
    cube = np.empty((len(cols), cfg.pixels, cfg.bands), dtype=np.float32)
    threads = threads or min(16, os.cpu_count() or 1)

    def work(j):
        c = cols[j]
        _fill_column(cfg, c, k, albedo[c], alpha[c], cube[j])

    if threads > 1 and len(cols) > 1:
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(work, range(len(cols))))
    else:
        for j in range(len(cols)):
            work(j)
    truth = {"alpha": alpha[cols], "albedo": albedo[cols]}
    return cube, unit_absorption(cfg), truth


def noiseless_scene(cols=2, pixels=400, bands=12, absorbing=6, frac=0.02, s0=-2e-4, seed=7,
                    albedo=1.0):
    """Separable noiseless scene for exact recovery.

    Box-shaped s (s0 < 0 on `absorbing` contiguous bands S, 0 elsewhere);
    L_i = a*(b + u_i) + alpha_i * a*(b (.) s) with u_i supported off S, exactly
    zero-mean over the background pixels and zero on plume pixels; constant
    albedo a. Returns (cube float32, s float32, truth alpha float64).
    The fp32 cube is built so that its exact fp64 promotion has the stated
    structure (u is zero-meaned after rounding to float32).
    """
    rng = _rng(seed, 99)
    s = np.zeros(bands, dtype=np.float32)
    j0 = (bands - absorbing) // 2
    S = np.arange(j0, j0 + absorbing)
    s[S] = np.float32(s0)
    off = np.setdiff1d(np.arange(bands), S)
    cube = np.empty((cols, pixels, bands), dtype=np.float32)
    truth = np.zeros((cols, pixels))
    m = int(round(frac * pixels))
    for c in range(cols):
        b = (2.0 + rng.uniform(0, 1, size=bands)).astype(np.float32)
        plume = rng.choice(pixels, size=m, replace=False)
        bg = np.setdiff1d(np.arange(pixels), plume)
        # integer-valued (in units of 2^-12) deviations so the fp32 values and
        # their background mean are exact
        u = np.zeros((pixels, bands))
        u_bg = rng.integers(-2048, 2049, size=(len(bg), len(off))).astype(np.float64)
        u_bg -= np.round(u_bg.mean(axis=0))[None, :]
        # make the column sums exactly zero: put the residual on the last pixel
        u_bg[-1] -= u_bg.sum(axis=0)
        u[np.ix_(bg, off)] = u_bg / 4096.0
        at = rng.uniform(500.0, 3000.0, size=m)
        truth[c, plume] = at
        base = albedo * (b.astype(np.float64)[None, :] + u)
        sig = np.zeros((pixels, bands))
        sig[plume] = at[:, None] * (albedo * b.astype(np.float64) * s.astype(np.float64))[None, :]
        cube[c] = (base + sig).astype(np.float32)
    return cube, s, truth
