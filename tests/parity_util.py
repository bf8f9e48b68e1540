"""Parity bar (BASELINE.json north_star):
|d alpha| <= 1e-3 * max|alpha_oracle| + 1 ppm m per pixel, relative albedo error
<= 1e-5; also reported: zero-set agreement, pixels beyond tolerance."""
import numpy as np

ALPHA_REL = 1e-3
ALPHA_ABS = 1.0
ALBEDO_REL = 1e-5


def compare(gpu_alpha, gpu_albedo, ora_alpha, ora_albedo, label=""):
    ga = np.asarray(gpu_alpha, np.float64)
    oa = np.asarray(ora_alpha, np.float64)
    fin = np.isfinite(oa)
    tol = ALPHA_REL * np.abs(oa[fin]).max(initial=0.0) + ALPHA_ABS
    diff = np.abs(ga - oa)
    bad = fin & ~(diff <= tol)
    nan_mismatch = np.isnan(ga) != np.isnan(oa)
    gr = np.asarray(gpu_albedo, np.float64)
    orr = np.asarray(ora_albedo, np.float64)
    finr = np.isfinite(orr)
    rel = np.abs(gr[finr] - orr[finr]) / np.maximum(np.abs(orr[finr]), 1e-30)
    zero_agree = ((ga[fin] == 0) == (oa[fin] == 0)).mean() if fin.any() else 1.0
    rep = dict(label=label, max_abs=float(diff[fin].max(initial=0.0)), tol=float(tol),
               n_bad=int(bad.sum()), n_nan_mismatch=int(nan_mismatch.sum()),
               albedo_max_rel=float(rel.max(initial=0.0)), zero_set_agreement=float(zero_agree),
               n=int(fin.sum()))
    return rep


def assert_parity(gpu_alpha, gpu_albedo, ora_alpha, ora_albedo, label=""):
    rep = compare(gpu_alpha, gpu_albedo, ora_alpha, ora_albedo, label)
    assert rep["n_nan_mismatch"] == 0, rep
    assert rep["n_bad"] == 0, rep
    assert rep["albedo_max_rel"] <= ALBEDO_REL, rep
    return rep


def c18_classify(gpu_alpha, ora_alpha, cube_col, s, run_oracle, tol, seeds=(1, 2)):
    """for pixels beyond tolerance, rerun the oracle with the
    input perturbed by +-1 fp32 ulp (random sign per element). Pixels whose
    perturbed oracle runs themselves move by more than the tolerance are
    ill-conditioned (reported separately); the others are real mismatches."""
    ga = np.asarray(gpu_alpha, np.float64)
    oa = np.asarray(ora_alpha, np.float64)
    bad = np.flatnonzero(~(np.abs(ga - oa) <= tol))
    if bad.size == 0:
        return dict(n_bad=0, ill_conditioned=[], well_conditioned=[])
    moved = np.zeros(bad.size, bool)
    for sd in seeds:
        rng = np.random.default_rng(sd)
        up = rng.random(cube_col.shape) < 0.5
        pert = np.where(up, np.nextafter(cube_col, np.float32(np.inf)),
                        np.nextafter(cube_col, np.float32(-np.inf))).astype(np.float32)
        ap = run_oracle(pert, s)
        moved |= np.abs(ap[bad] - oa[bad]) > tol
    return dict(n_bad=int(bad.size), ill_conditioned=[int(i) for i in bad[moved]],
                well_conditioned=[int(i) for i in bad[~moved]],
                gpu=[float(ga[i]) for i in bad], oracle=[float(oa[i]) for i in bad])
